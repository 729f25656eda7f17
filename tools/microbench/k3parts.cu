// Micro-benchmark of K3's per-vertex building blocks in isolation (one CTA,
// data already in shared memory): rank sorts (raw key / weight key), the
// serial lkk and suffix chains, fp64 division. clock64 around each part.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//          -I../../paper_2505_02977_b200/csrc/cuda k3parts.cu -o k3parts
#include <cstdio>
#include "../../paper_2505_02977_b200/csrc/cuda/eliminate.cu"

namespace parac_gpu {
void note_launches(long long) {}
}
using namespace parac_gpu;

__global__ void parts(int m, long long* out, double* sink) {
  __shared__ unsigned long long A[1024], X1[1024], X2[1024];
  __shared__ double B[1024], Cs[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) {
    A[i] = (static_cast<unsigned long long>((i * 2654435761u) & 0xfffff) << 32) | 1u;
    B[i] = 1.0 + ((i * 40503u) & 1023) * 1e-3;
  }
  __syncthreads();
  long long t0 = clock64();
  Scratch S{A, B, Cs, X1, X2};
  for (int rep = 0; rep < 10; ++rep) {
    unsigned long long wk[1], ak[1];
    const int g = tid;
    wk[0] = g < m ? dbits(B[g]) : kInfBits;
    ak[0] = g < m ? A[g] : ~0ull;
    int rank[1];
    rank_sort<kThreads, 1>(wk, m, S.X1, S.X2, reinterpret_cast<int*>(Cs), reinterpret_cast<int*>(Cs) + 1024, rank);
    __syncthreads();
    if (g < m) { X1[rank[0]] = ak[0]; }
    __syncthreads();
  }
  long long t1 = clock64();
  double s = 0;
  for (int rep = 0; rep < 10; ++rep) {
    if (tid == 0) s += serial_total(B, m);
    __syncthreads();
  }
  long long t2 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    if (tid == 0) serial_suffix(B, Cs, m);
    __syncthreads();
  }
  long long t3 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    for (int t = tid; t < m; t += blockDim.x) Cs[t] = __ddiv_rn(-B[t], 3.3 + rep);
    __syncthreads();
  }
  long long t4 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    unsigned long long key[1];
    key[0] = tid < m ? A[tid] : ~0ull;
    int rank[1];
    rank_sort<kThreads, 1>(key, m, S.X1, S.X2, reinterpret_cast<int*>(Cs), reinterpret_cast<int*>(Cs) + 1024, rank);
    if (tid < m) X2[rank[0]] = key[0];
    __syncthreads();
  }
  long long t5 = clock64();
  for (int rep = 0; rep < 10 && m <= kThreads; ++rep) {
    unsigned long long wk[1], ak[1];
    const int g = tid;
    wk[0] = g < m ? dbits(B[g]) : kInfBits;
    ak[0] = g < m ? A[g] : ~0ull;
    int rank[1];
    rank[0] = bcast_rank_cta<true>(wk[0], m, S.X2);
    __syncthreads();
    if (g < m) { X1[rank[0]] = ak[0]; }
    __syncthreads();
  }
  long long t6 = clock64();
  for (int rep = 0; rep < 10 && m <= kThreads; ++rep) {
    unsigned long long key[1];
    key[0] = tid < m ? A[tid] : ~0ull;
    int rank[1];
    rank[0] = bcast_rank_cta<false>(key[0], m, S.X1);
    __syncthreads();
    if (tid < m) X2[rank[0]] = key[0];
    __syncthreads();
  }
  long long t7 = clock64();
  if (tid == 0) {
    out[0] = (t1 - t0) / 10; out[1] = (t2 - t1) / 10; out[2] = (t3 - t2) / 10; out[3] = (t4 - t3) / 10;
    out[4] = (t5 - t4) / 10; out[5] = (t6 - t5) / 10; out[6] = (t7 - t6) / 10;
    sink[0] = s + Cs[3];
  }
}

__global__ void warp_parts(int m, long long* out) {
  __shared__ unsigned long long A[128], X1[128], X2[128];
  __shared__ double B[128], Cs[128];
  const int lane = threadIdx.x;
  for (int i = lane; i < 128; i += 32) {
    A[i] = (static_cast<unsigned long long>((i * 2654435761u) & 0xfffff) << 32) | 1u;
    B[i] = 1.0 + ((i * 40503u) & 1023) * 1e-3;
  }
  __syncwarp();
  Scratch S{A, B, Cs, X1, X2};
  long long t0 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    if (m <= 32) warp_rank_weight<1>(m, S, lane);
    else if (m <= 64) warp_rank_weight<2>(m, S, lane);
    else warp_rank_weight<4>(m, S, lane);
  }
  long long t1 = clock64();
  if (lane == 0) out[8] = (t1 - t0) / 10;
}


// cold-instruction-cache variant: one raw rank sort per launch (first touch of its code on that SM)
__global__ void cold_raw(int m, long long* out) {
  __shared__ unsigned long long A[1024], X1[1024], X2[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) A[i] = (static_cast<unsigned long long>((i * 2654435761u) & 0xfffff) << 32) | 1u;
  __syncthreads();
  long long t0 = clock64();
  unsigned long long key[1];
  key[0] = tid < m ? A[tid] : ~0ull;
  int rank[1];
  __shared__ int IAB[2048];
  rank_sort<kThreads, 1>(key, m, X1, X2, IAB, IAB + 1024, rank);
  if (tid < m) A[rank[0]] = key[0];
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[12 + blockIdx.x % 4] = t1 - t0;
}

int main() {
  long long* out; double* sink;
  cudaMalloc(&out, 256); cudaMalloc(&sink, 64);
  for (int m : {8, 32, 64, 103, 128, 200, 256}) {
    parts<<<1, kThreads>>>(m, out, sink);
    warp_parts<<<1, 32>>>(m <= 128 ? m : 128, out);
    long long h[16];
    cudaMemcpy(h, out, 128, cudaMemcpyDeviceToHost);
    printf("m=%3d  cta: weight rank sort %6lld  lkk chain %6lld  suffix chain %6lld  ddiv col %5lld  raw rank sort %6lld | bcast weight %6lld bcast raw %6lld cyc | warp weight sort (bcast) %6lld cyc\n",
           m, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[8]);
  }
  for (int m : {103, 173, 256}) {
    cold_raw<<<148, kThreads>>>(m, out);  // every SM runs the code once (cold)
    long long h[16];
    cudaMemcpy(h, out, 128, cudaMemcpyDeviceToHost);
    printf("cold raw rank sort m=%d: %lld %lld cycles (first touch per SM)\n", m, h[12], h[13]);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
