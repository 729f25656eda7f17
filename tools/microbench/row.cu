// Micro-benchmark: one warp computing one long sweep row (gather + products +
// serial subtraction), as in sweep_forward_kernel. Isolates service time.
#include <cstdio>
#include <cstdlib>
#include <vector>
constexpr int kRowBlock = 256;
__device__ __forceinline__ double serial_sub(double acc, const double* buf, int cnt) {
  int j = 0;
  for (; j + 8 <= cnt; j += 8) {
    double p[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) p[q] = buf[j + q];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = __dsub_rn(acc, p[q]);
  }
  for (; j < cnt; ++j) acc = __dsub_rn(acc, buf[j]);
  return acc;
}
__global__ void row(const int* col, const double* val, const double* yf, int len, double* out, long long* cyc) {
  __shared__ double wbuf[kRowBlock];
  const int lane = threadIdx.x;
  long long c0 = clock64();
  double acc = 1.0;
  for (int base = 0; base < len; base += kRowBlock) {
    const int cnt = min(kRowBlock, len - base);
// Stage the block: all index loads, then all value loads, then the products
    // (explicit register arrays: generic pointers would otherwise keep the
    // compiler from hoisting global loads above the shared-memory stores).
    int cidx[kRowBlock / 32];
    double yv[kRowBlock / 32], gv[kRowBlock / 32];
#pragma unroll
    for (int q = 0; q < kRowBlock / 32; ++q) cidx[q] = q * 32 + lane < cnt ? col[base + q * 32 + lane] : 0;
#pragma unroll
    for (int q = 0; q < kRowBlock / 32; ++q) {
      yv[q] = q * 32 + lane < cnt ? __ldcg(yf + cidx[q]) : 0.0;
      gv[q] = q * 32 + lane < cnt ? val[base + q * 32 + lane] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kRowBlock / 32; ++q)
      if (q * 32 + lane < cnt) wbuf[q * 32 + lane] = yv[q] != 0.0 ? __dmul_rn(gv[q], yv[q]) : 0.0;
    __syncwarp();
    if (lane == 0) acc = serial_sub(acc, wbuf, cnt);
    __syncwarp();
  }
  long long c1 = clock64();
  if (lane == 0) { out[0] = acc; cyc[0] = c1 - c0; }
}
int main() {
  const int N = 1 << 21;
  std::vector<int> hc(4096); std::vector<double> hv(4096), hy(N);
  for (int i = 0; i < 4096; ++i) { hc[i] = rand() % N; hv[i] = 1.0 / (i + 1); }
  for (int i = 0; i < N; ++i) hy[i] = 1.0 + (i % 7);
  int* c; double *v, *y, *o; long long* cy;
  cudaMalloc(&c, 4096 * 4); cudaMalloc(&v, 4096 * 8); cudaMalloc(&y, N * 8); cudaMalloc(&o, 8); cudaMalloc(&cy, 8);
  cudaMemcpy(c, hc.data(), 4096 * 4, cudaMemcpyHostToDevice); cudaMemcpy(v, hv.data(), 4096 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(y, hy.data(), N * 8, cudaMemcpyHostToDevice);
  for (int len : {32, 128, 256, 530, 1024}) {
    for (int rep = 0; rep < 2; ++rep) {
      row<<<1, 32>>>(c, v, y, len, o, cy); cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
      if (rep) printf("row len %4d: %6lld cycles = %.2f us\n", len, h, h / 1965.0);
    }
  }
  return 0;
}
