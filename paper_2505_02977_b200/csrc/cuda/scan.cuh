// Exclusive scan of non-negative int32 counts into an int64 offset array of
// length n+1 (out[n] = total). Three passes: per-tile sums, a single-CTA scan
// of the tile sums, per-tile rescan + offset. Used for the forward-CSR
// pointer (K1) and the CSC column pointer (K4).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace parac_gpu {
namespace dev {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ long long block_exclusive_scan(long long v, long long* smem,
                                                          long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    long long s = lane < nw ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) smem[lane] = s;
  }
  __syncthreads();
  const long long warp_prefix = warp > 0 ? smem[warp - 1] : 0;
  *total = smem[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

__global__ void scan_tile_sums(const int* __restrict__ in, long long n, long long* tile_sums) {
  __shared__ long long smem[32];
  const long long base = static_cast<long long>(blockIdx.x) * kScanTile;
  long long s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const long long t = base + static_cast<long long>(i) * kScanThreads + threadIdx.x;
    if (t < n) s += in[t];
  }
  long long total;
  block_exclusive_scan(s, smem, &total);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// Single CTA: exclusive scan of tile sums in place (any count).
__global__ void scan_tile_offsets(long long* tile_sums, long long tiles) {
  __shared__ long long smem[32];
  long long carry = 0;
  for (long long base = 0; base < tiles; base += blockDim.x) {
    const long long t = base + threadIdx.x;
    const long long v = t < tiles ? tile_sums[t] : 0;
    long long total;
    const long long ex = block_exclusive_scan(v, smem, &total);
    if (t < tiles) tile_sums[t] = carry + ex;
    carry += total;
  }
}

__global__ void scan_finish(const int* __restrict__ in, long long n,
                            const long long* __restrict__ tile_offsets, long long* out) {
  __shared__ long long smem[32];
  const long long base = static_cast<long long>(blockIdx.x) * kScanTile;
  // Each thread owns kScanItems consecutive elements (blocked arrangement).
  long long vals[kScanItems];
  long long s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const long long t = base + static_cast<long long>(threadIdx.x) * kScanItems + i;
    vals[i] = t < n ? in[t] : 0;
    s += vals[i];
  }
  long long total;
  long long run = block_exclusive_scan(s, smem, &total) + tile_offsets[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const long long t = base + static_cast<long long>(threadIdx.x) * kScanItems + i;
    if (t < n) out[t] = run;
    run += vals[i];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) out[n] = run;
}

}  // namespace dev
}  // namespace parac_gpu
