// Stable LSD radix sort of (key, int value) pairs, hand-written for the setup
// paths that need a deterministic order: the device ordering_nnz_sort
// (ordering.cu) and the solve layout's (level, position) order
// (solve_kernels.cu). Both are one-time, HBM-bound passes over n elements.
//
// One 8-bit digit per pass, three launches per pass:
//   tile_hist   one CTA per 4096-element tile, warp-aggregated shared counts,
//               written digit-major: counts[d * tiles + tile]
//   row_scan    one CTA per digit, exclusive scan of its per-tile counts in
//               place plus the digit total (the scatter CTAs scan the 256
//               totals themselves)
//   scatter     one CTA per tile; the tile is read in 16 rounds of 256, each
//               element ranked among equal digits by __match_any_sync inside
//               its warp plus the counts of the lower warps of the round, so
//               the output keeps input order within a digit (stability)
// Keys above end_bit must be zero (callers build them that way).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <string>

#include "../host/errors.hpp"

namespace parac_gpu {
void note_launches(long long k);  // defined in capi.cu
namespace radix {
namespace {  // internal linkage: each including unit gets its own kernels

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRounds = 16;
constexpr int kTile = kThreads * kRounds;

template <class K>
__device__ __forceinline__ unsigned digit_of(K k, int shift) {
  return static_cast<unsigned>(static_cast<unsigned long long>(k) >> shift) & 0xFFu;
}

template <class K>
__global__ void __launch_bounds__(kThreads) tile_hist_kernel(int n, const K* __restrict__ keys, int shift, int tiles,
                                                             unsigned* __restrict__ counts) {
  __shared__ unsigned h[256];
  const int t = threadIdx.x;
  h[t] = 0;
  __syncthreads();
  const long long base = static_cast<long long>(blockIdx.x) * kTile;
#pragma unroll 4
  for (int r = 0; r < kRounds; ++r) {
    const long long i = base + r * kThreads + t;
    const unsigned d = i < n ? digit_of(keys[i], shift) : 0x100u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (d < 256u && (peers & ((1u << (t & 31)) - 1u)) == 0u) atomicAdd(&h[d], static_cast<unsigned>(__popc(peers)));
  }
  __syncthreads();
  counts[static_cast<std::size_t>(t) * tiles + blockIdx.x] = h[t];
}

// Exclusive scan across one CTA of kThreads threads; *total gets the sum.
// ws: kWarps words of shared scratch (free again when this returns).
__device__ __forceinline__ unsigned block_excl_scan(unsigned x, unsigned* ws, unsigned* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    unsigned v = lane < kWarps ? ws[lane] : 0u;
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane < kWarps) ws[lane] = v;
  }
  __syncthreads();
  const unsigned r = (w ? ws[w - 1] : 0u) + inc - x;
  *total = ws[kWarps - 1];
  __syncthreads();
  return r;
}

// One CTA per digit: exclusive scan of that digit's per-tile counts in place
// (coalesced, 256 at a time); totals[d] = the digit's count over all tiles.
__global__ void __launch_bounds__(kThreads) row_scan_kernel(int tiles, unsigned* __restrict__ counts,
                                                            unsigned* __restrict__ totals) {
  __shared__ unsigned ws[kWarps];
  unsigned* row = counts + static_cast<std::size_t>(blockIdx.x) * tiles;
  unsigned carry = 0;
  for (int b = 0; b < tiles; b += kThreads) {
    const int i = b + threadIdx.x;
    const unsigned x = i < tiles ? row[i] : 0u;
    unsigned sum;
    const unsigned e = block_excl_scan(x, ws, &sum);
    if (i < tiles) row[i] = carry + e;
    carry += sum;
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

template <class K>
__global__ void __launch_bounds__(kThreads) scatter_kernel(int n, const K* __restrict__ kin, const int* __restrict__ vin,
                                                           K* __restrict__ kout, int* __restrict__ vout, int shift,
                                                           int tiles, const unsigned* __restrict__ offs,
                                                           const unsigned* __restrict__ totals) {
  __shared__ unsigned run[256];
  __shared__ unsigned wc[kWarps][256];
  __shared__ unsigned ws[kWarps];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  unsigned all;
  run[t] = block_excl_scan(totals[t], ws, &all) + offs[static_cast<std::size_t>(t) * tiles + blockIdx.x];
  const long long base = static_cast<long long>(blockIdx.x) * kTile;
  for (int r = 0; r < kRounds; ++r) {
#pragma unroll
    for (int j = 0; j < kWarps; ++j) wc[j][t] = 0;
    __syncthreads();
    const long long i = base + r * kThreads + t;
    const bool valid = i < n;
    K k{};
    int v = 0;
    unsigned d = 0x100u;
    if (valid) {
      k = kin[i];
      v = vin[i];
      d = digit_of(k, shift);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned lower = peers & ((1u << lane) - 1u);
    if (valid && lower == 0u) wc[w][d] = static_cast<unsigned>(__popc(peers));
    __syncthreads();
    if (valid) {
      unsigned pos = run[d] + static_cast<unsigned>(__popc(lower));
      for (int j = 0; j < w; ++j) pos += wc[j][d];
      kout[pos] = k;
      vout[pos] = v;
    }
    __syncthreads();
    unsigned s = 0;
#pragma unroll
    for (int j = 0; j < kWarps; ++j) s += wc[j][t];
    run[t] += s;
  }
}

inline void rs_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Failure{internal_error, std::string(what) + ": " + cudaGetErrorString(e)};
}

// Sorts the n pairs held in (k[0], v[0]) stably by key bits [0, end_bit),
// ping-ponging through (k[1], v[1]). Returns the index (0 or 1) of the buffers
// holding the result. Stream-ordered; no host synchronisation.
template <class K>
int sort_pairs(int n, K* k[2], int* v[2], int end_bit, cudaStream_t st) {
  if (n <= 1 || end_bit <= 0) return 0;
  const int tiles = (n + kTile - 1) / kTile;
  const long long total = 256LL * tiles;
  unsigned* counts = nullptr;
  rs_check(cudaMallocAsync(&counts, sizeof(unsigned) * static_cast<std::size_t>(total + 256), st), "radix alloc");
  unsigned* totals = counts + total;
  int cur = 0;
  for (int shift = 0; shift < end_bit; shift += 8) {
    tile_hist_kernel<K><<<tiles, kThreads, 0, st>>>(n, k[cur], shift, tiles, counts);
    row_scan_kernel<<<256, kThreads, 0, st>>>(tiles, counts, totals);
    scatter_kernel<K><<<tiles, kThreads, 0, st>>>(n, k[cur], v[cur], k[cur ^ 1], v[cur ^ 1], shift, tiles, counts,
                                                  totals);
    note_launches(3);
    cur ^= 1;
  }
  rs_check(cudaGetLastError(), "radix launch");
  rs_check(cudaFreeAsync(counts, st), "radix free");
  return cur;
}

}  // namespace
}  // namespace radix
}  // namespace parac_gpu
