// Micro-benchmark of the wide-column slab sort (eliminate.cu slab_sort) on ONE
// CTA in isolation: R unique raw keys in a global slab, 40 KB of dynamic shared
// memory for the tile scratch, globaltimer around the call. Compare with the
// in-situ numbers of tools/profile_factor.py (wide_columns).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//          slabsort.cu -o slabsort
#include <cstdio>
#include <vector>
#include <cub/block/block_radix_sort.cuh>
#include "../../paper_2505_02977_b200/csrc/cuda/eliminate.cu"

namespace parac_gpu {
void note_launches(long long) {}
}
using namespace parac_gpu;

template <typename Less>
__global__ void run(unsigned long long* K, unsigned long long* V, unsigned long long* K2, unsigned long long* V2,
                    int R, unsigned long long padk, unsigned long long* out) {
  extern __shared__ char smem[];
  const XBuf sxb{reinterpret_cast<unsigned long long*>(smem), reinterpret_cast<unsigned long long*>(smem + 8 * kBigCap),
                 reinterpret_cast<unsigned long long*>(smem + 3 * 8 * kBigCap),
                 reinterpret_cast<unsigned long long*>(smem + 4 * 8 * kBigCap)};
  unsigned long long tiles = 0;
  for (int rep = 0; rep < 3; ++rep) {  // rep 0: cold instruction cache; reps 1-2: warm
    __syncthreads();
    const unsigned long long t0 = globaltimer_ns();
    slab_sort(K, V, K2, V2, R, padk, 0ull, sxb, Less{}, threadIdx.x == 0 ? &tiles : nullptr);
    const unsigned long long t1 = globaltimer_ns();
    if (threadIdx.x == 0) {
      out[2 * rep] = t1 - t0;
      out[2 * rep + 1] = tiles - t0;
    }
  }
}


// rank_sort<kThreads, 4> alone on shared-memory data (no global traffic), 10 reps
__global__ void rank_only(unsigned long long* out, int R) {
  extern __shared__ char smem[];
  unsigned long long* X1 = reinterpret_cast<unsigned long long*>(smem);
  unsigned long long* X2 = X1 + 1024;
  int* IA = reinterpret_cast<int*>(X2 + 1024);
  int* IB = IA + 1024;
  unsigned long long key[4];
  for (int i = 0; i < 4; ++i) {
    const unsigned g = i * kThreads + threadIdx.x;
    key[i] = (static_cast<unsigned long long>((g * 2654435761u) % 4000000u) << 32) | (g + 1);
  }
  int rank[4];
  __shared__ long long cyc[3];
  __syncthreads();
  const long long c0 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    rank_sort<kThreads, 4>(key, R, X1, X2, IA, IB, rank, cyc);
    __syncthreads();
  }
  const long long c1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (c1 - c0) / 10;
    out[1] = cyc[0];
    out[2] = cyc[1];
    out[3] = cyc[2];
  }
}

int main() {
  const int Rs[] = {1024, 2048, 4096, 5600, 16384, 65536};
  unsigned long long *K, *V, *K2, *V2, *out;
  const int cap = 1 << 17;
  cudaMalloc(&K, cap * 8); cudaMalloc(&V, cap * 8); cudaMalloc(&K2, cap * 8); cudaMalloc(&V2, cap * 8);
  cudaMalloc(&out, 48);
  cudaFuncSetAttribute(run<RawLess>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCtaSmem);
  cudaFuncSetAttribute(run<WeightLess>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCtaSmem);
  for (int R : Rs) {
    std::vector<unsigned long long> k(R), v(R);
    for (int i = 0; i < R; ++i) {
      const unsigned long long row = (static_cast<unsigned long long>(i) * 2654435761ull) % 4000000ull;
      k[i] = (row << 32) | static_cast<unsigned>(i + 1);
      v[i] = i;
    }
    for (int which = 0; which < 2; ++which) {
      unsigned long long best = ~0ull, bt = 0;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemcpy(K, k.data(), R * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(V, v.data(), R * 8, cudaMemcpyHostToDevice);
        if (which == 0) run<RawLess><<<1, kThreads, kCtaSmem>>>(K, V, K2, V2, R, ~0ull, out);
        else run<WeightLess><<<1, kThreads, kCtaSmem>>>(K, V, K2, V2, R, ~0ull, out);
        unsigned long long h[6];
        cudaMemcpy(h, out, 48, cudaMemcpyDeviceToHost);
        if (rep == 0) printf("   cold %.1f us (tiles %.1f) warm %.1f us (tiles %.1f)\n", h[0] / 1e3, h[1] / 1e3,
                             h[4] / 1e3, h[5] / 1e3);
        if (h[4] < best) { best = h[4]; bt = h[5]; }
      }
      std::vector<unsigned long long> r(R);
      cudaMemcpy(r.data(), K, R * 8, cudaMemcpyDeviceToHost);
      bool ok = true;
      for (int i = 1; i < R; ++i) ok &= r[i - 1] <= r[i];
      printf("R %6d %s: total %8.1f us, tiles %8.1f us, merges %8.1f us %s\n", R, which ? "weight" : "raw   ",
             best / 1e3, bt / 1e3, (best - bt) / 1e3, ok ? "sorted" : "NOT SORTED");
    }
  }
  cudaFuncSetAttribute(rank_only, cudaFuncAttributeMaxDynamicSharedMemorySize, kCtaSmem);
  for (int R : {256, 512, 1024}) {
    rank_only<<<1, kThreads, kCtaSmem>>>(out, R);
    unsigned long long h[4];
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    printf("rank_sort<256,4> alone, R %d: %llu cycles (stage %llu, phase1 %llu, phase2 %llu)\n", R, h[0], h[1],
           h[2], h[3]);
  }
  const cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
