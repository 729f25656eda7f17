// The hub path's serial FP64 chains in isolation (cycles per element):
// lkk-style left-to-right sum and suffix (right to left, outputs stored),
// from shared memory, alone and side by side on two warps.
#include <cstdio>
__device__ __forceinline__ double chain_sum(double s, const double* x, int cnt) {
  int t = 0;
  for (; t + 8 <= cnt; t += 8) {
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = x[t + q];
#pragma unroll
    for (int q = 0; q < 8; ++q) s = __dadd_rn(s, a[q]);
  }
  for (; t < cnt; ++t) s = __dadd_rn(s, x[t]);
  return s;
}
__device__ __forceinline__ double chain_suffix(double s, const double* x, double* o, int cnt) {
  int g = cnt - 1;
  for (; g >= 7; g -= 8) {
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = x[g - q];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      s = __dadd_rn(a[q], s);
      o[g - q] = s;
    }
  }
  for (; g >= 0; --g) {
    s = __dadd_rn(x[g], s);
    o[g] = s;
  }
  return s;
}
__device__ __forceinline__ double chain_suffix_sfirst(double s, const double* x, double* o, int cnt) {
  int g = cnt - 1;
  for (; g >= 7; g -= 8) {
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = x[g - q];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      s = __dadd_rn(s, a[q]);
      o[g - q] = s;
    }
  }
  for (; g >= 0; --g) {
    s = __dadd_rn(s, x[g]);
    o[g] = s;
  }
  return s;
}
__global__ void k(const double* in, int n, int mode, double* out, long long* cyc) {
  __shared__ double X[2048], O[2048];
  for (int i = threadIdx.x; i < n; i += blockDim.x) X[i] = in[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long c0 = clock64();
  double s = 0;
  if (lane == 0) {
    if (mode == 0 && warp == 0) s = chain_sum(0.0, X, n);
    if (mode == 1 && warp == 1) s = chain_suffix(0.0, X, O, n);
    if (mode == 3 && warp == 1) s = chain_suffix_sfirst(0.0, X, O, n);
    if (mode == 2 && warp == 0) s = chain_sum(0.0, X, n);
    if (mode == 2 && warp == 1) s = chain_suffix(0.0, X, O, n);
  }
  long long c1 = clock64();
  if (lane == 0 && warp < 2) {
    out[warp] = s + O[7];
    cyc[warp] = c1 - c0;
  }
}
int main() {
  double *in, *out;
  long long* cyc;
  const int n = 2048;
  cudaMallocManaged(&in, n * 8);
  cudaMallocManaged(&out, 16);
  cudaMallocManaged(&cyc, 16);
  for (int i = 0; i < n; ++i) in[i] = 1.0 / (i + 1);
  const char* names[4] = {"sum alone", "suffix alone", "both (warp 0 sum, warp 1 suffix)", "suffix, sum as first operand"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cyc[0] = cyc[1] = 0;
      k<<<1, 256>>>(in, n, mode, out, cyc);
      cudaDeviceSynchronize();
    }
    printf("%-36s warp0 %.2f  warp1 %.2f cycles/element\n", names[mode], cyc[0] / double(n), cyc[1] / double(n));
  }
  return 0;
}
