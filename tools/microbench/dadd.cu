// Dependent FP64 add latency on one thread (the exact PCG's serial chains):
// cycles per __dadd_rn in a chain fed from shared memory, 1 and 2 interleaved chains.
#include <cstdio>
__global__ void chain(const double* in, int n, int reps, double* out, long long* cyc) {
  __shared__ double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = in[i];
  __syncthreads();
  if (threadIdx.x) return;
  double s = 0, t = 0;
  long long c0 = clock64();
  for (int r = 0; r < reps; ++r)
    for (int i = 0; i < 4096; i += 8) {
      double u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) u[q] = buf[i + q];
#pragma unroll
      for (int q = 0; q < 8; ++q) s = __dadd_rn(s, u[q]);
    }
  long long c1 = clock64();
  for (int r = 0; r < reps; ++r)
    for (int i = 0; i < 4096; i += 8) {
      double u[8], v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) { u[q] = buf[i + q]; v[q] = buf[4095 - i - q]; }
#pragma unroll
      for (int q = 0; q < 8; ++q) { s = __dadd_rn(s, u[q]); t = __dadd_rn(t, v[q]); }
    }
  long long c2 = clock64();
  out[0] = s + t;
  cyc[0] = c1 - c0;
  cyc[1] = c2 - c1;
}
int main() {
  double *in, *out; long long* cyc;
  cudaMallocManaged(&in, 4096 * 8); cudaMallocManaged(&out, 8); cudaMallocManaged(&cyc, 16);
  for (int i = 0; i < 4096; ++i) in[i] = 1.0 / (i + 1);
  const int reps = 64;
  chain<<<1, 128>>>(in, 4096, reps, out, cyc);
  cudaDeviceSynchronize();
  const double adds = 4096.0 * reps;
  printf("one chain: %.2f cycles/add; two interleaved chains: %.2f cycles per add-pair\n", cyc[0] / adds, cyc[1] / adds);
  return 0;
}
