// Device helpers shared by the factorization kernels (K1-K4).
#pragma once
#include "common.cuh"
#include "factor_kernels.cuh"

namespace parac_gpu {
namespace fdev {

using namespace dev;

constexpr double kDropThreshold = 1e-300;  // factor_common.hpp:149
constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;
enum : int { kErrArena = 10, kErrStall = 11, kErrPerm = 8, kErrInternal = 17, kErrNeedHubs = kStatusNeedHubs };

__device__ __forceinline__ void fail(const FactorDev& d, int code, long long info) {
  if (atomicCAS(&d.ctrl->status, 0, code) == 0) d.ctrl->err_info = info;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned long long dbits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}
__device__ __forceinline__ double bitsd(unsigned long long x) {
  return __longlong_as_double(static_cast<long long>(x));
}

__device__ __forceinline__ int next_pow2(int x) { return x <= 1 ? 1 : 1 << (32 - __clz(x - 1)); }

// TestHooks::delay analogue: pseudo-random __nanosleep at phase boundaries.
__device__ __forceinline__ void maybe_delay(const FactorDev& d, int k, int phase) {
  if (d.delay_ns > 0) {
    const unsigned long long h = mix64(static_cast<unsigned long long>(k) * 4 + phase);
    if (h % 5 == 0) __nanosleep(static_cast<unsigned>(h % static_cast<unsigned>(d.delay_ns)));
  }
}

// Fill-slot addressing (see factor_kernels.cuh). Chunk c >= 1 of slot s.
struct SlotLoc {
  int c;          // 0 = preallocated first chunk
  long long off;  // offset inside the chunk
};
__device__ __forceinline__ SlotLoc slot_loc(int c0, int s) {
  if (s < c0) return {0, s};
  const unsigned q = static_cast<unsigned>(s / c0) + 1u;
  const int c = 31 - __clz(q);
  return {c, s - static_cast<long long>(c0) * ((1ll << c) - 1)};
}

// Address of fill slot s of position lo for READING (the chunk is known to be
// allocated: every writer finished before lo became ready).
__device__ __forceinline__ const int4* fill_slot_read(const FactorDev& d, int lo, int s) {
  if (s < d.c0) return d.pool0 + static_cast<long long>(lo) * d.c0 + s;
  const SlotLoc L = slot_loc(d.c0, s);
  const unsigned e = static_cast<unsigned>(
      ld_relaxed(reinterpret_cast<const int*>(d.dir + static_cast<long long>(lo) * kDirChunks + L.c - 1)));
  return d.ovf + static_cast<long long>(e - 1) * d.c0 + L.off;
}

// Raw entry t of column k: forward edge (source -1 -> key low word 0) or fill.
__device__ __forceinline__ void load_raw(const FactorDev& d, int k, long long fb, int fdeg, int t,
                                         unsigned long long& key, double& w) {
  if (t < fdeg) {
    key = static_cast<unsigned long long>(static_cast<unsigned>(__ldg(d.fwd_to + fb + t))) << 32;
    w = __ldg(d.fwd_w + fb + t);
  } else {
    const int4 e = ld_cg_int4(fill_slot_read(d, k, t - fdeg));
    key = (static_cast<unsigned long long>(static_cast<unsigned>(e.x)) << 32) |
          static_cast<unsigned>(e.y + 1);
    w = __hiloint2double(e.w, e.z);
  }
}

// load_raw with the column's fill directory row prefetched (dirrow[c-1] =
// chunk c's directory entry): one dependent round trip less per entry.
__device__ __forceinline__ void load_raw_dir(const FactorDev& d, int k, long long fb, int fdeg, int t,
                                             const unsigned* dirrow, unsigned long long& key,
                                             double& w) {
  if (t < fdeg) {
    key = static_cast<unsigned long long>(static_cast<unsigned>(__ldg(d.fwd_to + fb + t))) << 32;
    w = __ldg(d.fwd_w + fb + t);
    return;
  }
  const int s = t - fdeg;
  const int4* src;
  if (s < d.c0) {
    src = d.pool0 + static_cast<long long>(k) * d.c0 + s;
  } else {
    const SlotLoc L = slot_loc(d.c0, s);
    src = d.ovf + static_cast<long long>(dirrow[L.c - 1] - 1) * d.c0 + L.off;
  }
  const int4 e = ld_cg_int4(src);
  key = (static_cast<unsigned long long>(static_cast<unsigned>(e.x)) << 32) |
        static_cast<unsigned>(e.y + 1);
  w = __hiloint2double(e.w, e.z);
}

// Reserve fill slot for (lo) and allocate its overflow chunk if this slot is
// the chunk's first. Returns the slot, or -1 on budget exhaustion.
__device__ __forceinline__ int reserve_fill_slot(const FactorDev& d, int lo) {
  const int slot = static_cast<int>(atomicAdd(&d.cnt[lo], 1ull << 32) >> 32);
  if (slot >= d.c0) {
    const SlotLoc L = slot_loc(d.c0, slot);
    if (L.c > kDirChunks) {
      fail(d, kErrArena, lo);
      return -1;
    }
    if (L.off == 0) {
      const unsigned long long sz = static_cast<unsigned long long>(d.c0) << L.c;
      const unsigned long long at = atomicAdd(&d.ctrl->ovf_bump, sz);
      if (static_cast<long long>(at + sz) > d.ovf_cap) {
        fail(d, kErrArena, lo);
        return -1;
      }
      // Writers of the chunk only need its address (no data hand-off): relaxed.
      asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(d.dir + static_cast<long long>(lo) * kDirChunks + L.c - 1),
                   "r"(static_cast<unsigned>(at / d.c0) + 1u)
                   : "memory");
    }
  }
  return slot;
}

// Write a fill into a reserved slot (spins while another writer allocates the chunk).
__device__ __forceinline__ bool write_fill(const FactorDev& d, int lo, int slot, int hi, int src,
                                           double w) {
  int4* dst;
  if (slot < d.c0) {
    dst = d.pool0 + static_cast<long long>(lo) * d.c0 + slot;
  } else {
    const SlotLoc L = slot_loc(d.c0, slot);
    const int* de = reinterpret_cast<const int*>(d.dir + static_cast<long long>(lo) * kDirChunks + L.c - 1);
    unsigned e = static_cast<unsigned>(ld_relaxed(de));
    while (e == 0) {
      if (ld_relaxed(&d.ctrl->status) != 0) return false;
      __nanosleep(32);
      e = static_cast<unsigned>(ld_relaxed(de));
    }
    dst = d.ovf + static_cast<long long>(e - 1) * d.c0 + L.off;
  }
  const long long wb = __double_as_longlong(w);
  st_cg_int4(dst, make_int4(hi, src, static_cast<int>(wb & 0xffffffffll), static_cast<int>(wb >> 32)));
  return true;
}

// The fills a column received are read exactly once, by its own gather, and
// no writer touches the column's preallocated slots after it became ready:
// drop those L2 lines without a write-back (the next factorization rewrites
// every slot before it is read). Slots [0, min(fc, c0)) of position k, lines
// t, t + step, ...
__device__ __forceinline__ void discard_fills(const FactorDev& d, int k, int fc, int t, int step) {
  if (!d.discard_fills) return;
  const long long bytes = 16ll * min(fc, d.c0);
  const char* base = reinterpret_cast<const char*>(d.pool0 + static_cast<long long>(k) * d.c0);
  for (long long off = 128ll * t; off < bytes; off += 128ll * step)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + off) : "memory");
}

// pick_by_suffix (include/parac/sampling.hpp:46-57)
__device__ __forceinline__ int pick_by_suffix(const double* suffix, int lo, int hi, double u) {
  while (lo < hi) {
    const int mid = lo + (hi - lo + 1) / 2;
    if (suffix[mid] > u) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// One sample of sample_clique_sorted (include/parac/sampling.hpp:77-83): the
// pair (v_i, v_j) and weight (s * w_i) / lkk. Returns false if dropped.
// Sampling stream of position k: (derived seed, key). A batch factors several
// independent problems as one disjoint union; each keeps its own seed and its
// own positions as keys, so every problem's factor equals its stand-alone one.
struct SampleKey {
  unsigned long long seed;
  long long key;
};
__device__ __forceinline__ SampleKey sample_key(const FactorDev& d, int k) {
  if (!d.pos_pid) return {d.sample_seed, k};
  const int p = d.pos_pid[k];
  return {d.pid_seed[p], static_cast<long long>(k) - d.pid_base[p]};
}

// pick_by_suffix over a wide column: coarse index (every kCoarse-th suffix
// value, shared memory) then a fine search in global memory. Same result as
// the flat search: suffix is non-increasing, so {j : suffix[j] > u} is a prefix.
constexpr int kCoarse = 64;        // minimum coarse step
constexpr int kCoarseMax = 2048;   // coarse entries (16 KB of shared memory)
__device__ __forceinline__ int coarse_step(int m) { return max(kCoarse, (m + kCoarseMax - 1) / kCoarseMax); }
__device__ __forceinline__ int pick_wide(const double* suffix, const double* coarse, int cs, int lo, int hi,
                                         double u) {
  // largest coarse point q*cs inside [lo, hi] with suffix > u, then the fine search after it
  int qlo = (lo + cs - 1) / cs, qhi = hi / cs;
  int a = lo;
  if (qlo <= qhi && coarse[qlo] > u) {
    while (qlo < qhi) {
      const int mid = qlo + (qhi - qlo + 1) / 2;
      if (coarse[mid] > u) qlo = mid; else qhi = mid - 1;
    }
    a = max(lo, qlo * cs);
  }
  const int b = min(hi, a + cs);
  return pick_by_suffix(suffix, a, b, u);
}

__device__ __forceinline__ bool draw_sample(const FactorDev& d, SampleKey sk, int k, int i, int m,
                                           const unsigned long long* A, const double* B,
                                           const double* suffix, double lkk, int& lo, int& hi,
                                           double& wv, const double* coarse = nullptr, int cs = 0) {
  const double s = suffix[i + 1];
  const double u = __dmul_rn(unit_uniform(sk.seed, sk.key, static_cast<unsigned long long>(i)), s);
  const int j = coarse ? pick_wide(suffix, coarse, cs, i + 1, m - 1, u) : pick_by_suffix(suffix, i + 1, m - 1, u);
  wv = __ddiv_rn(__dmul_rn(s, B[i]), lkk);
  if (wv < kDropThreshold) return false;
  const int a = static_cast<int>(A[i] >> 32), c = static_cast<int>(A[j] >> 32);
  lo = min(a, c);
  hi = max(a, c);
  return true;
}

// Publish (warp-aggregated) the rows of lanes with pub set to the big queue
// when big, else to the main queue. The caller has already issued a release
// fence, so relaxed stores suffice (they pair with the consumer's relaxed poll
// + acquire fence).
__device__ __forceinline__ void publish(const FactorDev& d, bool pub, bool big, int row, int lane) {
  const unsigned bm = __ballot_sync(kFull, pub && !big);
  const unsigned bb = __ballot_sync(kFull, pub && big);
  if ((bm | bb) == 0) return;
  int qm = 0, qb = 0;
  if (lane == 0) {
    if (bm) qm = atomicAdd(&d.ctrl->q_tail, __popc(bm));
    if (bb) qb = atomicAdd(&d.ctrl->b_tail, __popc(bb));
  }
  qm = __shfl_sync(kFull, qm, 0);
  qb = __shfl_sync(kFull, qb, 0);
  if (pub) {
    int* slot = big ? &d.bqueue[qb + __popc(bb & lanemask_lt())]
                    : &d.queue[qm + __popc(bm & lanemask_lt())];
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(slot), "r"(row) : "memory");
  }
}

}  // namespace fdev
}  // namespace parac_gpu
