// Micro-benchmarks calibrating the per-vertex cost model of K3 on B200:
// serial DADD chain (smem-fed), warp register bitonic (32 x u64+f64),
// CTA hybrid bitonic (256 x 2 x u64), globaltimer resolution.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void dadd_chain(double* out, long long* cyc, int m) {
  __shared__ double B[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) B[i] = 1.0 + i * 1e-3;
  __syncthreads();
  if (threadIdx.x) return;
  long long c0 = clock64();
  double s = 0.0;
  for (int rep = 0; rep < 10; ++rep) {
    int i = 0;
    for (; i + 4 <= m; i += 4) { double x0=B[i],x1=B[i+1],x2=B[i+2],x3=B[i+3]; s=__dadd_rn(s,x0); s=__dadd_rn(s,x1); s=__dadd_rn(s,x2); s=__dadd_rn(s,x3);}
    for (; i < m; ++i) s = __dadd_rn(s, B[i]);
  }
  long long c1 = clock64();
  out[0] = s; cyc[0] = (c1 - c0) / 10;
}

__global__ void warp_sort32(unsigned long long* out, long long* cyc) {
  const int lane = threadIdx.x & 31;
  unsigned long long key = (lane * 2654435761u) & 0xffff; double val = lane;
  long long c0 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      unsigned long long pk = __shfl_xor_sync(~0u, key, j); double pv = __shfl_xor_sync(~0u, val, j);
      bool lower = (lane & j) == 0, up = (lane & k) == 0;
      bool take = (lower == up) ? (pk < key) : (pk > key);
      key = take ? pk : key; val = take ? pv : val;
    }
    key ^= rep;
  }
  long long c1 = clock64();
  out[lane] = key + (unsigned long long)val;
  if (lane == 0) cyc[1] = (c1 - c0) / 10;
}

__global__ void cta_sort256(unsigned long long* out, long long* cyc) {
  __shared__ unsigned long long K0[256], V0[256], K1[256], V1[256];
  const int tid = threadIdx.x, lane = tid & 31;
  unsigned long long key = (tid * 2654435761u) & 0xfffff, val = tid;
  __syncthreads();
  long long c0 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    int buf = 0;
#pragma unroll
    for (int k = 2; k <= 256; k <<= 1)
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        unsigned long long pk, pv; bool lower;
        if (j < 32) { pk = __shfl_xor_sync(~0u, key, j); pv = __shfl_xor_sync(~0u, val, j); lower = (lane & j) == 0; }
        else { unsigned long long* KB = buf ? K1 : K0; unsigned long long* VB = buf ? V1 : V0;
               KB[tid] = key; VB[tid] = val; __syncthreads(); pk = KB[tid ^ j]; pv = VB[tid ^ j]; lower = (tid & j) == 0; buf ^= 1; }
        bool up = (tid & k) == 0;
        bool take = (lower == up) ? (pk < key) : (pk > key);
        key = take ? pk : key; val = take ? pv : val;
      }
    key ^= rep;
  }
  long long c1 = clock64();
  out[tid] = key + val;
  if (tid == 0) cyc[2] = (c1 - c0) / 10;
}

__global__ void timer_res(long long* cyc) {
  unsigned long long t0 = gt(), t1;
  int changes = 0; unsigned long long last = t0, mind = ~0ull;
  long long c0 = clock64();
  while (changes < 20) { t1 = gt(); if (t1 != last) { if (t1 - last < mind) mind = t1 - last; last = t1; ++changes; } }
  long long c1 = clock64();
  cyc[3] = mind; cyc[4] = (c1 - c0) / 20; cyc[5] = (last - t0) / 20;
}

__global__ void l2_atomic_rt(int* p, long long* cyc) {
  long long c0 = clock64();
  int v = 0;
  for (int i = 0; i < 100; ++i) v += atomicAdd(p + (v & 1) * 64, 1);
  long long c1 = clock64();
  cyc[6] = (c1 - c0) / 100; cyc[15] = v;
  c0 = clock64();
  for (int i = 0; i < 100; ++i) { __threadfence(); v += atomicAdd(p, 1); }
  c1 = clock64();
  cyc[7] = (c1 - c0) / 100;
  volatile int* vp = p + 256;
  c0 = clock64();
  for (int i = 0; i < 100; ++i) v += vp[v & 7];
  c1 = clock64();
  cyc[8] = (c1 - c0) / 100; cyc[14] = v;
}

int main() {
  double* od; unsigned long long* ou; long long* cyc; int* ai;
  cudaMalloc(&od, 8); cudaMalloc(&ou, 4096); cudaMalloc(&cyc, 16 * 8); cudaMalloc(&ai, 8192);
  cudaMemset(ai, 0, 8192); cudaMemset(cyc, 0, 128);
  for (int m : {16, 64, 128, 256}) {
    dadd_chain<<<1, 128>>>(od, cyc, m); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dadd chain m=%d: %lld cycles (%.2f cyc/add)\n", m, h, (double)h / m);
  }
  warp_sort32<<<1, 32>>>(ou, cyc); cta_sort256<<<1, 256>>>(ou, cyc); timer_res<<<1, 1>>>(cyc);
  l2_atomic_rt<<<1, 1>>>(ai, cyc);
  cudaDeviceSynchronize();
  long long h[16]; cudaMemcpy(h, cyc, 128, cudaMemcpyDeviceToHost);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("warp bitonic 32 (u64+f64): %lld cycles\ncta hybrid bitonic 256: %lld cycles\n", h[1], h[2]);
  printf("globaltimer min step %lld ns, %lld cycles/change, %lld ns/change\n", h[3], h[4], h[5]);
  printf("atomicAdd RT %lld cyc, fence+atomic %lld cyc, volatile load RT %lld cyc; clock %d kHz\n", h[6], h[7], h[8], clk);
  return 0;
}
