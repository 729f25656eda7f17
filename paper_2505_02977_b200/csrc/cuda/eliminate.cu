// K3: the persistent elimination kernel (sm_100a).
//
// One elimination = factor_sequential's loop body (proj/src/factor_seq.cpp:70-138)
// with the par-backends' dependency hand-off (proj/src/factor_par.cpp:282-293,
// 424-477); SURVEY Appendix A steps 1-9:
//   gather (forward edges ++ fills) -> sort by (row, source) -> merge runs
//   (serial sums) -> lkk (serial) -> column -> sort by (weight, row) -> suffix
//   (serial, right to left) -> sample + emit fills (dp[hi]++) -> fence ->
//   decrement dp[row] by multiplicity -> rows reaching zero are ready.
//
// Work split. Persistent CTAs of 8 warps, two roles:
//   * small CTAs: every warp eliminates its own vertex, raw size R <= kSmallCap,
//     sorted entirely in registers (bitonic network over 32*ITEMS elements);
//   * big CTAs (every 4th): the whole CTA eliminates one vertex with
//     R <= kBigCap in shared memory (256-thread bitonic networks); wider
//     columns use a global slab.
// A vertex that becomes ready is routed by its final R to the main or the big
// ready queue. The warp/CTA that makes vertices ready keeps the widest one it
// can hold and eliminates it next without a queue round trip (keep-one): the
// critical path runs through exactly these hand-offs.
//
// Bit-exactness: the serial sums use __dadd_rn in the reference's order, the
// products/divisions __dmul_rn/__ddiv_rn; sort keys are unique, so any sorting
// network reproduces the reference's order.
#include "k3_common.cuh"

#include <algorithm>

namespace parac_gpu {

void note_launches(long long k);

using namespace dev;
using namespace fdev;
using namespace k3;

namespace {

constexpr int kBatch = (kSmallCap + 31) / 32;  // samples / decrements per lane in flight (small path): one batch

// Role of this CTA. On a full grid the role follows the SM (every 4th SM runs
// only big CTAs) so each SM executes a single code path and its instruction
// cache holds one path's working set; tiny grids (tests) fall back to CTA ids.
__device__ __forceinline__ bool is_big_cta() {
  if (gridDim.x < 148) return (blockIdx.x & 3) == 3 || blockIdx.x == gridDim.x - 1;
  unsigned smid;
  asm("mov.u32 %0, %%smid;" : "=r"(smid));
  return (smid & 3) == 3;
}

// Column scratch views. A: raw key (row << 32 | source+1), then merged
// (row << 32 | multiplicity); B: weights; C: suffix sums, then the ready list.
struct Scratch {
  unsigned long long* A;
  double* B;
  double* C;
  unsigned long long* X1;  // rank-sort sorted-segment buffers (shared-memory scratch only)
  unsigned long long* X2;
};
__device__ __forceinline__ Scratch carve(char* base, int cap) {
  return {reinterpret_cast<unsigned long long*>(base),
          reinterpret_cast<double*>(base + 8 * static_cast<long long>(cap)),
          reinterpret_cast<double*>(base + 16 * static_cast<long long>(cap)),
          reinterpret_cast<unsigned long long*>(base + 24 * static_cast<long long>(cap)),
          reinterpret_cast<unsigned long long*>(base + 32 * static_cast<long long>(cap))};
}

// What the keeper already knows about the vertex it keeps.
struct Next {
  int k;        // vertex, -1 none
  int fdeg;     // forward degree (-1: unknown)
  int fc;       // fills received
  long long fb; // forward-CSR offset
};

// ------------------------------------------------------------ claiming
// Claim the next slot of a ready queue and spin on it (relaxed polls, backoff
// by distance to the tail). Returns the vertex, -1 when every vertex is
// eliminated, -2 on abort. The caller issues the acquire fence.
// claim_at waits on slot idx; with help != nullptr (big CTAs) it also watches
// the latest posted hub job (Ctrl::hub_hint) and returns -3 (job in *help)
// when it has chunks left, keeping the slot for later.
__device__ __forceinline__ int claim_at(const FactorDev& d, bool big, int idx, int* help) {
  int* queue = big ? d.bqueue : d.queue;
  if (idx >= d.n) return -1;
  int v = ld_relaxed(&queue[idx]);
  if (v >= 0) return v;
  unsigned long long t0 = globaltimer_ns();
  int last = ld_relaxed(&d.ctrl->eliminated);
  int iter = 0;
  unsigned ns = 32;
  while (true) {
    // Distance probe on a slot-specific address (no shared word polled by
    // every waiter): if the slot 16 places earlier is still empty, we are far
    // from the publishing front and sleep long. Probes are dependent round
    // trips, so they run on every 8th poll only.
    if ((iter & 7) == 0 || ns >= 512) {  // long sleepers re-probe every time
      if (idx < 16 || ld_relaxed(&queue[idx - 16]) >= 0) ns = 32;
      else if (idx < 256 || ld_relaxed(&queue[idx - 256]) >= 0) ns = d.sleep_ns[0];
      else if (idx < 1024 || ld_relaxed(&queue[idx - 1024]) >= 0) ns = d.sleep_ns[1];
      else ns = d.sleep_ns[2];  // far waiters must not load the L2
    }
    if (help) {  // a posted hub phase with chunks left: go and help
      ns = min(ns, d.hub_wait_ns);  // a new hub job must find helpers within its first phase
      const int hj = ld_relaxed(&d.ctrl->hub_hint);
      if (hj > 0) {
        const unsigned long long nx = ld_relaxed_u64(&d.hub_jobs[hj - 1].next);
        if ((nx & 0xffffffull) < ((nx >> 24) & 0xffffffull)) {
          *help = hj - 1;
          return -3;
        }
        ns = min(ns, 64u);  // the next phase of an active job follows within microseconds
      }
    }
    __nanosleep(ns);
    v = ld_relaxed(&queue[idx]);
    if (v >= 0) return v;
    if ((++iter & 15) == 0) {
      if (ld_relaxed(&d.ctrl->status) != 0) return -2;
      const int done = ld_relaxed(&d.ctrl->eliminated);
      if (done >= d.n) return -1;
      const unsigned long long now = globaltimer_ns();
      if (done != last) {
        last = done;
        t0 = now;
      } else if (now - t0 > d.watchdog_ns) {
        fail(d, kErrStall, idx);
        return -2;
      }
    }
  }
}

__device__ __forceinline__ int claim(const FactorDev& d, bool big) {
  return claim_at(d, big, atomicAdd(big ? &d.ctrl->b_head : &d.ctrl->q_head, 1), nullptr);
}

// ------------------------------------------------------------ sorting
// (weight bits, A) strictly-less: fill_sorted_view order (factor_common.hpp:140-144);
// A = row << 32 | mult and rows are unique, so the multiplicity never decides.
__device__ __forceinline__ bool wless(unsigned long long wa, unsigned long long aa,
                                      unsigned long long wb, unsigned long long ab) {
  return wa < wb || (wa == wb && aa < ab);
}

// ------------------------------------------------------------ sorting networks
// All networks sort (key, val) u64 pairs ascending under Less (keys are unique
// under Less). Stage loops are runtime loops on purpose: fully unrolled
// networks made K3 ~0.5 MB of SASS and the critical path instruction-fetch
// bound (measured).

struct RawLess {  // unique raw keys; the payload (weight bits) never decides
  __device__ __forceinline__ bool operator()(unsigned long long a, unsigned long long,
                                             unsigned long long b, unsigned long long) const {
    return a < b;
  }
};
struct WeightLess {  // key = weight bits, val = row << 32 | mult
  __device__ __forceinline__ bool operator()(unsigned long long wa, unsigned long long aa,
                                             unsigned long long wb, unsigned long long ab) const {
    return wless(wa, aa, wb, ab);
  }
};

// Compare-exchange of items i < p held by one thread (ascending if up).
template <typename Less>
__device__ __forceinline__ void cx(unsigned long long& ki, unsigned long long& vi,
                                   unsigned long long& kp, unsigned long long& vp, bool up, Less less) {
  const bool sw = less(kp, vp, ki, vi) == up;
  const unsigned long long k0 = sw ? kp : ki, k1 = sw ? ki : kp;
  const unsigned long long v0 = sw ? vp : vi, v1 = sw ? vi : vp;
  ki = k0;
  kp = k1;
  vi = v0;
  vp = v1;
}

// Intra-thread stage (distance j < ITEMS <= 4), element g = base + i.
template <int ITEMS, typename Less>
__device__ __forceinline__ void intra_stage(unsigned long long (&key)[ITEMS],
                                            unsigned long long (&val)[ITEMS], int base, int k, int j,
                                            Less less) {
  if constexpr (ITEMS >= 2) {
    if (j == 1) {
#pragma unroll
      for (int i = 0; i < ITEMS; i += 2) cx(key[i], val[i], key[i + 1], val[i + 1], ((base + i) & k) == 0, less);
    }
  }
  if constexpr (ITEMS >= 4) {
    if (j == 2) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i)
        if ((i & 2) == 0) cx(key[i], val[i], key[i + 2], val[i + 2], ((base + i) & k) == 0, less);
    }
  }
}

// Cross-lane stage through shuffles: partner lane = lane ^ lm.
template <int ITEMS, typename Less>
__device__ __forceinline__ void shfl_stage(unsigned long long (&key)[ITEMS],
                                           unsigned long long (&val)[ITEMS], int base, int k, int lm,
                                           bool lower, Less less) {
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const unsigned long long pk = __shfl_xor_sync(kFull, key[i], lm);
    const unsigned long long pv = __shfl_xor_sync(kFull, val[i], lm);
    const bool up = ((base + i) & k) == 0;
    const bool take = (lower == up) ? less(pk, pv, key[i], val[i]) : less(key[i], val[i], pk, pv);
    key[i] = take ? pk : key[i];
    val[i] = take ? pv : val[i];
  }
}

// Warp register bitonic sort of 32*ITEMS elements, blocked layout
// (element g = lane*ITEMS + i).
template <int ITEMS, typename Less>
__device__ __forceinline__ void warp_reg_sort(unsigned long long (&key)[ITEMS],
                                           unsigned long long (&val)[ITEMS], int lane, Less less) {
  constexpr int P = 32 * ITEMS;
  const int base = lane * ITEMS;
#pragma unroll 1
  for (int k = 2; k <= P; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < ITEMS) intra_stage<ITEMS>(key, val, base, k, j, less);
      else shfl_stage<ITEMS>(key, val, base, k, j / ITEMS, (lane & (j / ITEMS)) == 0, less);
    }
  }
}

// Hybrid CTA bitonic network over P = 256*ITEMS elements in registers
// (element g = tid*ITEMS + i): intra-thread, then shuffles, and stages wider
// than a warp exchange through shared memory, double-buffered (striped layout
// i*256 + tid, conflict-free), one barrier per such stage.
struct XBuf {
  unsigned long long* k0;
  unsigned long long* v0;
  unsigned long long* k1;
  unsigned long long* v1;
};

template <int ITEMS, typename Less>
__device__ __forceinline__ void cta_reg_sort(unsigned long long (&key)[ITEMS],
                                          unsigned long long (&val)[ITEMS], XBuf xb, Less less) {
  constexpr int P = kThreads * ITEMS;
  const int tid = threadIdx.x, lane = tid & 31;
  const int base = tid * ITEMS;
  int buf = 0;
#pragma unroll 1
  for (int k = 2; k <= P; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < ITEMS) {
        intra_stage<ITEMS>(key, val, base, k, j, less);
      } else if (j < 32 * ITEMS) {
        shfl_stage<ITEMS>(key, val, base, k, j / ITEMS, (lane & (j / ITEMS)) == 0, less);
      } else {
        const int tm = j / ITEMS;
        unsigned long long* KB = buf ? xb.k1 : xb.k0;
        unsigned long long* VB = buf ? xb.v1 : xb.v0;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          KB[i * kThreads + tid] = key[i];
          VB[i * kThreads + tid] = val[i];
        }
        __syncthreads();
        const int pt = tid ^ tm;
        const bool lower = (tid & tm) == 0;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const unsigned long long pk = KB[i * kThreads + pt];
          const unsigned long long pv = VB[i * kThreads + pt];
          const bool up = ((base + i) & k) == 0;
          const bool take = (lower == up) ? less(pk, pv, key[i], val[i]) : less(key[i], val[i], pk, pv);
          key[i] = take ? pk : key[i];
          val[i] = take ? pv : val[i];
        }
        buf ^= 1;
      }
    }
  }
}


// ------------------------------------------------------------ rank sort
// Stable sort of R <= T*ITEMS u64 keys held in registers (element g = i*T +
// tid; ties keep g order), T = 32 (one warp) or kThreads (the CTA). Two
// phases, branch-free compares, broadcast shared-memory reads:
//   1. rank inside the element's 32-element segment (32 broadcast loads of
//      the unsorted keys, staged in X2); the segment is written sorted to X1;
//   2. add, for every other segment, how many of its keys precede the
//      element (5-step binary search of the sorted segment: keys <= k for
//      earlier segments, < k for later ones -- that is the stable tie rule).
// Raw keys (row << 32 | source+1) are unique. The weight sort needs (weight,
// row) order; its input is already row-ascending, so a STABLE sort on the
// weight bits alone gives exactly fill_sorted_view's order
// (factor_common.hpp:133-145).
// All-pairs stable rank with broadcast shared-memory reads: element g of the
// R keys gets
//   rank = #{t : X[t] < k_g} + (STABLE ? #{t < g : X[t] == k_g} : 0)
// (raw keys are unique; the weight sort needs the stable tie rule). One
// barrier, broadcast 16-byte loads and four independent compare/accumulate
// chains per element: no dependent binary-search rounds, no barriers per
// round. The stable rule is free outside the 32-key block holding g's own
// warp: keys before that block count when <= k (compare against k + 1),
// keys after it when < k; inside it the threshold switches at g.

// Warp: element g = i*32 + lane of R <= 32*ITEMS; block b holds keys
// [32b, 32b+32), item i's own block is b == i (compile-time).
template <int ITEMS, bool STABLE>
__device__ __forceinline__ void bcast_rank_warp(const unsigned long long (&k)[ITEMS], int R, unsigned long long* X,
                                                int (&rank)[ITEMS]) {
  const int lane = lane_id();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i)
    if (i * 32 + lane < R) X[i * 32 + lane] = k[i];
  if (lane == 0 && (R & 1)) X[R] = ~0ull;
  __syncwarp();
  const ulonglong2* X2 = reinterpret_cast<const ulonglong2*>(X);
  int ca[ITEMS], cb[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) ca[i] = cb[i] = 0;
#pragma unroll 1
  for (int b = 0; b * 32 < R; ++b) {
    const ulonglong2* P = X2 + 16 * b;
    const int pairs = (min(32, R - 32 * b) + 1) >> 1;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (STABLE && i == b) count_below_mixed(P, pairs, k[i], lane, ca[i], cb[i]);
      else count_below(P, 0, pairs, STABLE && i > b ? k[i] + 1 : k[i], ca[i], cb[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) rank[i] = ca[i] + cb[i];
}

// ---- warp path (rank sort): gather + raw sort, weight sort (results in A/B)
template <int ITEMS>
__device__ __forceinline__ void warp_rank_raw(const FactorDev& d, int k, long long fb, int fdeg, int R,
                                              Scratch S, int lane, unsigned long long* stamp) {
  unsigned long long key[ITEMS], val[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = i * 32 + lane;
    key[i] = ~0ull;
    val[i] = 0;
    if (g < R) {
      double w;
      load_raw(d, k, fb, fdeg, g, key[i], w);
      val[i] = dbits(w);
    }
  }
  if (stamp && lane == 0) {  // diagnostics: the lead's gather has landed
    asm volatile("" ::"l"(key[0]), "l"(val[0]));
    *stamp = globaltimer_ns();
  }
  int rank[ITEMS];
  bcast_rank_warp<ITEMS, false>(key, R, S.X1, rank);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (i * 32 + lane < R) {
      S.A[rank[i]] = key[i];
      S.B[rank[i]] = bitsd(val[i]);
    }
  }
  __syncwarp();
}

template <int ITEMS>
__device__ __forceinline__ void warp_rank_weight(int m, Scratch S, int lane) {
  unsigned long long wk[ITEMS], ak[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = i * 32 + lane;
    wk[i] = g < m ? dbits(S.B[g]) : kInfBits;
    ak[i] = g < m ? S.A[g] : ~0ull;
  }
  int rank[ITEMS];
  bcast_rank_warp<ITEMS, true>(wk, m, S.X1, rank);
  __syncwarp();  // every lane has read A/B
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (i * 32 + lane < m) {
      S.A[rank[i]] = ak[i];
      S.B[rank[i]] = bitsd(wk[i]);
    }
  }
  __syncwarp();
}

// ---- CTA path (rank sort), R <= kThreads * ITEMS
template <int ITEMS>
__device__ __forceinline__ void cta_rank_raw(const FactorDev& d, int k, long long fb, int fdeg, int R,
                                             const unsigned* dirrow, Scratch S, unsigned long long* stamp) {
  unsigned long long key[ITEMS], val[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = i * kThreads + threadIdx.x;
    key[i] = ~0ull;
    val[i] = 0;
    if (g < R) {
      double w;
      load_raw_dir(d, k, fb, fdeg, g, dirrow, key[i], w);
      val[i] = dbits(w);
    }
  }
  if (stamp) {  // diagnostics: every thread's gather has landed
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) asm volatile("" ::"l"(key[i]), "l"(val[i]));
    __syncthreads();
    if (threadIdx.x == 0) *stamp = globaltimer_ns();
  }
  int rank[ITEMS];
  long long* cyc = d.vsub ? reinterpret_cast<long long*>(d.vsub + d.n * 8ll + 4ll * k) : nullptr;
  if constexpr (ITEMS == 1) {
    (void)cyc;
    rank[0] = bcast_rank_cta<false>(key[0], R, S.X1);
  } else {
    rank_sort<kThreads, ITEMS>(key, R, S.X1, S.X2, reinterpret_cast<int*>(S.C), reinterpret_cast<int*>(S.C) + kBigCap, rank, cyc);
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (i * kThreads + static_cast<int>(threadIdx.x) < R) {
      S.A[rank[i]] = key[i];
      S.B[rank[i]] = bitsd(val[i]);
    }
  }
  __syncthreads();
}

// ---- CTA path: gather + merge by hashing (R <= kBigCap), no raw sort.
// factor_common.hpp:100-113 sorts the raw column by (row, source) and sums
// each row's run left to right. Only two orders matter for the bits: rows
// ascending (the merged column) and sources ascending inside a row (the
// summation order). So: hash the raw entries by row (shared-memory open
// addressing + a per-row list), let every entry count the entries of its row
// with a smaller key (its place in the run; sources are unique per row, see
// DESIGN.md), stage each run contiguously in that order, let the run's first
// entry sum it serially, then rank the m distinct rows with 32-bit broadcast
// compares. Output: merged (row << 32 | multiplicity, sum) in row order in
// (X1, X2). Returns m, or -1 when a row's run is longer than kRunCap (then the
// caller falls back to the full raw sort).
constexpr int kRunCap = 64;
template <int ITEMS>
__device__ __forceinline__ int cta_hash_merge(const FactorDev& d, int k, long long fb, int fdeg, int R,
                                              const unsigned* dirrow, Scratch S, CtaShared& sh,
                                              unsigned long long* stamp) {
  const int tid = threadIdx.x;
  int* tab = reinterpret_cast<int*>(S.X1);   // slot -> row, then slot -> stage base
  int* head = reinterpret_cast<int*>(S.X2);  // slot -> last pushed entry
  int* nxt = reinterpret_cast<int*>(S.C);    // entry -> next entry of its row
  int* rows32 = nxt + kBigCap;               // distinct rows (unordered)
  double* stage = S.B;                       // runs, contiguous, source order
  const int hbits = 32 - __clz(max(2 * R - 1, 1));  // table of 2^hbits >= 2R slots
  const int hs = 1 << hbits;
  unsigned long long key[ITEMS];
  double w[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = i * kThreads + tid;
    key[i] = ~0ull;
    w[i] = 0.0;
    if (g < R) load_raw_dir(d, k, fb, fdeg, g, dirrow, key[i], w[i]);
  }
  for (int t = tid; t < hs; t += kThreads) {
    tab[t] = -1;
    head[t] = -1;
  }
  if (tid == 0) {
    sh.mbump = 0;
    sh.mcount = 0;
    sh.hbad = 0;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = i * kThreads + tid;
    if (g < R) S.A[g] = key[i];
  }
  if (stamp) {  // diagnostics: every thread's gather has landed
    __syncthreads();
    if (tid == 0) *stamp = globaltimer_ns();
  }
  __syncthreads();
  // diagnostics (record_times): clock64 at the step barriers, 4 slots per position
  long long* cyc = stamp && tid == 0 ? reinterpret_cast<long long*>(d.vsub + d.n * 8ll + 4ll * k) : nullptr;
  const long long c0 = cyc ? clock64() : 0;
  // insert: slot of the row, push the entry on the row's list
  int slot[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = i * kThreads + tid;
    slot[i] = -1;
    if (g < R) {
      const int row = static_cast<int>(key[i] >> 32);
      int h = static_cast<int>((static_cast<unsigned>(row) * 0x9E3779B1u) >> (32 - hbits));
      while (true) {
        const int old = atomicCAS(&tab[h], -1, row);
        if (old == -1 || old == row) break;
        h = (h + 1) & (hs - 1);
      }
      slot[i] = h;
      nxt[g] = atomicExch(&head[h], g);
    }
  }
  __syncthreads();
  if (cyc) cyc[0] = clock64() - c0;
  // place in the run = entries of the row with a smaller key; run length
  int pos[ITEMS], len[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    pos[i] = 0;
    len[i] = 0;
    if (slot[i] >= 0) {
      int h = head[slot[i]];
      while (h >= 0 && len[i] <= kRunCap) {
        pos[i] += static_cast<int>(S.A[h] < key[i]);
        ++len[i];
        h = nxt[h];
      }
      if (len[i] > kRunCap) sh.hbad = 1;
    }
  }
  __syncthreads();  // every walk done: tab (rows) is free; hbad visible
  if (cyc) cyc[1] = clock64() - c0;
  if (sh.hbad) return -1;
  // stage base and compact index of each run: warp-level exclusive scans of
  // the run heads' lengths and counts, one shared-memory atomic per warp each
  int jj[ITEMS];
  {
    const int lane = tid & 31;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const bool headr = slot[i] >= 0 && pos[i] == 0;
      const int v = headr ? len[i] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned hm = __ballot_sync(kFull, headr);
      int base = 0, jb = 0;
      if (lane == 31 && hm) {
        base = atomicAdd(&sh.mbump, incl);
        jb = atomicAdd(&sh.mcount, __popc(hm));
      }
      base = __shfl_sync(kFull, base, 31);
      jb = __shfl_sync(kFull, jb, 31);
      jj[i] = jb + __popc(hm & lanemask_lt());
      if (headr) tab[slot[i]] = base + incl - v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i)
    if (slot[i] >= 0) stage[tab[slot[i]] + pos[i]] = w[i];
  __syncthreads();
  // run heads: serial sum in source order (merge_raw); (row, length, sum)
  // go to slot j of compact arrays (rows32, nxt, head as doubles: all free now)
  double* sumj = reinterpret_cast<double*>(head);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (slot[i] >= 0 && pos[i] == 0) {
      const double* st = stage + tab[slot[i]];
      double acc = st[0];
      for (int q = 1; q < len[i]; ++q) acc = __dadd_rn(acc, st[q]);
      const int j = jj[i];
      rows32[j] = static_cast<int>(key[i] >> 32);
      nxt[j] = len[i];
      sumj[j] = acc;
    }
  }
  __syncthreads();
  const int m = sh.mcount;
  if (cyc) cyc[2] = clock64() - c0;
  // rank of each distinct row (all-pairs, 32-bit, 4 rows per broadcast load),
  // spread over every thread; results written after a barrier (the output
  // overwrites the compact arrays)
  const int4* R4 = reinterpret_cast<const int4*>(rows32);
  const int quads = m >> 2;
  int rk[ITEMS], rrow[ITEMS], rlen[ITEMS];
  double rsum[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int j = i * kThreads + tid;
    rk[i] = -1;
    if (j < m) {
      const int row = rows32[j];
      int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll 4
      for (int q = 0; q < quads; ++q) {
        const int4 v = R4[q];
        c0 += static_cast<int>(v.x < row);
        c1 += static_cast<int>(v.y < row);
        c2 += static_cast<int>(v.z < row);
        c3 += static_cast<int>(v.w < row);
      }
      for (int t = 4 * quads; t < m; ++t) c0 += static_cast<int>(rows32[t] < row);
      rk[i] = c0 + c1 + c2 + c3;
      rrow[i] = row;
      rlen[i] = nxt[j];
      rsum[i] = sumj[j];
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (rk[i] >= 0) {
      S.X1[rk[i]] = (static_cast<unsigned long long>(static_cast<unsigned>(rrow[i])) << 32) |
                    static_cast<unsigned>(rlen[i]);
      reinterpret_cast<double*>(S.X2)[rk[i]] = rsum[i];
    }
  }
  __syncthreads();
  if (cyc) cyc[3] = clock64() - c0;
  return m;
}

template <int ITEMS>
__device__ __forceinline__ void cta_rank_weight(int m, Scratch S) {
  unsigned long long wk[ITEMS], ak[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = i * kThreads + threadIdx.x;
    wk[i] = g < m ? dbits(S.B[g]) : kInfBits;
    ak[i] = g < m ? S.A[g] : ~0ull;
  }
  int rank[ITEMS];
  if constexpr (ITEMS == 1) rank[0] = bcast_rank_cta<true>(wk[0], m, S.X1);
  else rank_sort<kThreads, ITEMS>(wk, m, S.X1, S.X2, reinterpret_cast<int*>(S.C), reinterpret_cast<int*>(S.C) + kBigCap, rank);
  __syncthreads();  // every thread has read A/B
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (i * kThreads + static_cast<int>(threadIdx.x) < m) {
      S.A[rank[i]] = ak[i];
      S.B[rank[i]] = bitsd(wk[i]);
    }
  }
  __syncthreads();
}

// ---- warp path: gather + raw sort, weight sort (results in A/B, natural order)
template <int ITEMS>
__device__ __forceinline__ void warp_sort_raw(const FactorDev& d, int k, long long fb, int fdeg,
                                              int R, Scratch S, int lane) {
  unsigned long long key[ITEMS], val[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = lane * ITEMS + i;
    key[i] = ~0ull;
    val[i] = 0;
    if (g < R) {
      double w;
      load_raw(d, k, fb, fdeg, g, key[i], w);
      val[i] = dbits(w);
    }
  }
  warp_reg_sort<ITEMS>(key, val, lane, RawLess{});
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    S.A[lane * ITEMS + i] = key[i];
    S.B[lane * ITEMS + i] = bitsd(val[i]);
  }
}

template <int ITEMS>
__device__ __forceinline__ void warp_sort_weight(int m, Scratch S, int lane) {
  unsigned long long wk[ITEMS], ak[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = lane * ITEMS + i;
    wk[i] = g < m ? dbits(S.B[g]) : kInfBits;
    ak[i] = g < m ? S.A[g] : ~0ull;
  }
  __syncwarp();
  warp_reg_sort<ITEMS>(wk, ak, lane, WeightLess{});
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    S.A[lane * ITEMS + i] = ak[i];
    S.B[lane * ITEMS + i] = bitsd(wk[i]);
  }
}

// ---- CTA path
template <int ITEMS>
__device__ __forceinline__ void cta_gather_sort_raw(const FactorDev& d, int k, long long fb, int fdeg,
                                                    int R, const unsigned* dirrow,
                                                    unsigned long long* A, double* B, XBuf xb) {
  unsigned long long key[ITEMS], val[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = threadIdx.x * ITEMS + i;
    key[i] = ~0ull;
    val[i] = 0;
    if (g < R) {
      double w;
      load_raw_dir(d, k, fb, fdeg, g, dirrow, key[i], w);
      val[i] = dbits(w);
    }
  }
  cta_reg_sort<ITEMS>(key, val, xb, RawLess{});
  __syncthreads();  // exchange buffers alias A/B
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    A[threadIdx.x * ITEMS + i] = key[i];
    B[threadIdx.x * ITEMS + i] = bitsd(val[i]);
  }
  __syncthreads();
}

template <int ITEMS>
__device__ __forceinline__ void cta_sort_weight_reg(int m, unsigned long long* A, double* B, XBuf xb) {
  unsigned long long wk[ITEMS], ak[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = threadIdx.x * ITEMS + i;
    wk[i] = g < m ? dbits(B[g]) : kInfBits;
    ak[i] = g < m ? A[g] : ~0ull;
  }
  __syncthreads();  // exchange buffers alias A/B
  cta_reg_sort<ITEMS>(wk, ak, xb, WeightLess{});
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    A[threadIdx.x * ITEMS + i] = ak[i];
    B[threadIdx.x * ITEMS + i] = bitsd(wk[i]);
  }
  __syncthreads();
}

// ------------------------------------------------------------ serial chains
// lkk = ((0 + w0) + w1) + ... in row order (factor_common.hpp:117-121)
__device__ __forceinline__ double serial_total(const double* B, int m) {
  double s = 0.0;
  int i = 0;
  for (; i + 8 <= m; i += 8) {
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = B[i + q];
#pragma unroll
    for (int q = 0; q < 8; ++q) s = __dadd_rn(s, x[q]);
  }
  for (; i < m; ++i) s = __dadd_rn(s, B[i]);
  return s;
}

// suffix[g] = w[g] + suffix[g+1], strictly right to left (sampling.hpp:72-76)
__device__ __forceinline__ void serial_suffix(const double* B, double* C, int m) {
  double s = B[m - 1];
  C[m - 1] = s;
  int g = m - 2;
  // loads of the next block are independent of the chain; stores after it
  // (C may alias nothing in B, but the compiler cannot know)
  for (; g >= 7; g -= 8) {
    double x[8], o[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = B[g - q];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      s = __dadd_rn(x[q], s);
      o[q] = s;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) C[g - q] = o[q];
  }
  for (; g >= 0; --g) {
    s = __dadd_rn(B[g], s);
    C[g] = s;
  }
}

// keep-one preference among the vertices an elimination made ready (max key
// wins; the low word is the row): the widest column, or (keep_pos) the lowest
// position -- the head of the longest remaining dependency chain.
__device__ __forceinline__ unsigned long long keep_key(const FactorDev& d, unsigned long long rr) {
  const unsigned row = static_cast<unsigned>(rr & 0xffffffffu);
  return d.keep_pos ? (1ull << 63) | (static_cast<unsigned long long>(0x7fffffffu - row) << 32) | row
                    : rr | (1ull << 63);
}

// ============================================================ small path
// One warp eliminates k (R <= kSmallCap). Returns the kept vertex, -1, or -2.
__device__ Next warp_eliminate(const FactorDev& d, Next nx, Scratch S, int lane, bool allow_keep) {
  const int k = nx.k;
  const bool lead = lane == 0;
  Ctrl* ctrl = d.ctrl;
  if (d.verify && lead && dp_of(ld_relaxed_u64(&d.cnt[k])) != 0) fail(d, kErrInternal, k);
  maybe_delay(d, k, 0);

  // ---- 1. gather
  long long fb = nx.fb;
  int fdeg = nx.fdeg, fc = nx.fc;
  if (fdeg < 0) {
    fb = d.fwd_ptr[k];
    fdeg = static_cast<int>(d.fwd_ptr[k + 1] - fb);
    fc = static_cast<int>(ld_relaxed_u64(&d.cnt[k]) >> 32);
  }
  const int R = fdeg + fc;
  // level[k] is final once k is ready (every predecessor raised it before its
  // releasing decrement); load it now, use it after the sampling phase
  const int lvk = d.level ? ld_relaxed(&d.level[k]) : 0;
  if (R > d.small_cap) {  // mis-routed (cannot happen with exact routing): hand to a big CTA
    publish(d, lead, true, k, lane);
    return {-3, -1, 0, 0};
  }
  long long start = 0;
  if (lead && R > 0)
    start = static_cast<long long>(atomicAdd(&ctrl->arena_bump, static_cast<unsigned long long>(R)));
  SUB(0);

  // ---- 2. sort raw by (row, source)  (factor_common.hpp:100-104), in registers
  if (R <= 32) warp_rank_raw<1>(d, k, fb, fdeg, R, S, lane, d.vsub ? d.vsub + 8 * static_cast<long long>(k) + 1 : nullptr);
  else if (R <= 64) warp_rank_raw<2>(d, k, fb, fdeg, R, S, lane, d.vsub ? d.vsub + 8 * static_cast<long long>(k) + 1 : nullptr);
  else warp_rank_raw<kBatch>(d, k, fb, fdeg, R, S, lane, d.vsub ? d.vsub + 8 * static_cast<long long>(k) + 1 : nullptr);
  __syncwarp();
  discard_fills(d, k, R - fdeg, lane, 32);
  PHASE(1);
  if (k == d.trace_k) snapshot_dp(d, 0, lane, 32);

  // ---- 3. merge runs in place: left-to-right sums, multiplicity = run length
  //      (factor_common.hpp:105-113). Chunk c writes only below 32(c+1).
  int m = 0;
  int carry_row = -1;
  for (int base = 0; base < R; base += 32) {
    const int t = base + lane;
    const int row = t < R ? static_cast<int>(S.A[t] >> 32) : -2;
    int prev = __shfl_up_sync(kFull, row, 1);
    if (lane == 0) prev = carry_row;
    const bool head = t < R && row != prev;
    double acc = 0.0;
    int c = 0;
    if (head) {
      acc = S.B[t];
      c = 1;
      while (t + c < R && static_cast<int>(S.A[t + c] >> 32) == row) {
        acc = __dadd_rn(acc, S.B[t + c]);
        ++c;
      }
    }
    carry_row = __shfl_sync(kFull, row, 31);
    const unsigned b = __ballot_sync(kFull, head);
    __syncwarp();
    if (head) {
      const int idx = m + __popc(b & lanemask_lt());
      S.A[idx] = (static_cast<unsigned long long>(static_cast<unsigned>(row)) << 32) |
                 static_cast<unsigned>(c);
      S.B[idx] = acc;
    }
    m += __popc(b);
    __syncwarp();
  }
  PHASE(2);
  if (m == 0) {  // factor_seq.cpp:92-95 (col_len/col_start already 0 from K1)
    if (lead) {
      d.diag[k] = 0.0;
      if (d.blk_done) fence_acq_rel();  // release: the streamed assembly reads it after the count
    }
    return {-1, -1, 0, 0};
  }

  // ---- 5. lkk + column k: rows ascending, values (-w)/lkk (factor_seq.cpp:97-102)
  double lkk = lead ? serial_total(S.B, m) : 0.0;
  lkk = __shfl_sync(kFull, lkk, 0);
  start = __shfl_sync(kFull, start, 0);
  if (start + m > d.arena_cap) {
    if (lead) fail(d, kErrArena, k);
    return {-2, -1, 0, 0};
  }
  for (int t = lane; t < m; t += 32) {
    d.arena_rows[start + t] = static_cast<int>(S.A[t] >> 32);
    d.arena_vals[start + t] = __ddiv_rn(-S.B[t], lkk);
  }
  if (lead) {
    d.diag[k] = lkk;
    d.col_start[k] = start;
    d.col_len[k] = m;
  }
  PHASE(3);

  // ---- 6-7. weight sort (registers) + suffix
  if (m >= 2) {
    if (m <= 32) warp_rank_weight<1>(m, S, lane);
    else if (m <= 64) warp_rank_weight<2>(m, S, lane);
    else warp_rank_weight<kBatch>(m, S, lane);
    __syncwarp();
    SUB(2);
    if (lead) serial_suffix(S.B, S.C, m);
    __syncwarp();
  }
  PHASE(4);

  // ---- 8. sampling + fill emission (m - 1 <= 127 samples: one batch)
  const SampleKey sk = sample_key(d, k);
  int emitted = 0;
  bool bad = false;
  {
    bool em[kBatch];
    int lo[kBatch], hi[kBatch], slot[kBatch];
    double wv[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int i = b * 32 + lane;
      em[b] = i < m - 1 && draw_sample(d, sk, k, i, m, S.A, S.B, S.C, lkk, lo[b], hi[b], wv[b]);
    }
    SUB(3);
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      if (em[b]) {
        slot[b] = reserve_fill_slot(d, lo[b]);
        red_add_relaxed_u64(&d.cnt[hi[b]], 1ull);
        bad = bad || slot[b] < 0;
      }
    }
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      if (em[b] && !bad) bad = !write_fill(d, lo[b], slot[b], hi[b], k, wv[b]);
      emitted += __popc(__ballot_sync(kFull, em[b]));
    }
  }
  SUB(4);
  if (__any_sync(kFull, bad)) return {-2, -1, 0, 0};
  if (lead) d.samples[k] = emitted;
  // ASAP level of the factor DAG (schedule_levels, factor_par.cpp:659-684):
  // level[row] >= level[k] + 1, published before the decrements release row.
  if (d.level) {
    const int lk = lvk + 1;
    for (int t = lane; t < m; t += 32) atomicMax(&d.level[static_cast<int>(S.A[t] >> 32)], lk);
  }
  PHASE(5);
  maybe_delay(d, k, 1);

  // ---- 9. release every emission, then decrement (factor_par.cpp:282-293)
  fence_acq_rel();
  __syncwarp();
  SUB(5);
  if (k == d.trace_k) snapshot_dp(d, 1, lane, 32);
  unsigned long long* ready = reinterpret_cast<unsigned long long*>(S.C);
  int nready = 0;
  {
    int row[kBatch], mult[kBatch], fd[kBatch];
    unsigned long long old[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int t = b * 32 + lane;
      row[b] = -1;
      mult[b] = fd[b] = 0;
      old[b] = 0;
      if (t < m) {
        const unsigned long long a = S.A[t];
        row[b] = static_cast<int>(a >> 32);
        mult[b] = static_cast<int>(a & 0xffffffffu);
        fd[b] = __ldg(&d.fdeg[row[b]]);  // in flight with the decrement
        old[b] = atom_add_relaxed_u64(&d.cnt[row[b]], static_cast<unsigned long long>(-static_cast<long long>(mult[b])));
      }
    }
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      if (d.verify && row[b] >= 0 && dp_of(old[b]) < mult[b]) fail(d, kErrInternal, row[b]);
      // no fence here: whoever eliminates a ready vertex acquires first (loop top / claim)
      const bool now_ready = row[b] >= 0 && dp_of(old[b]) == mult[b];
      const unsigned bm = __ballot_sync(kFull, now_ready);
      if (now_ready) ready[nready + __popc(bm & lanemask_lt())] = ready_info(row[b], fd[b], old[b]);
      nready += __popc(bm);
    }
  }
  __syncwarp();
  PHASE(6);
  if (k == d.trace_k) snapshot_dp(d, 2, lane, 32);
  maybe_delay(d, k, 2);
  if (nready == 0) return {-1, -1, 0, 0};

  // keep-one: the best ready column this warp can hold (lowest position by
  // default); publish the rest
  unsigned long long best = 0;
  for (int t = lane; t < nready; t += 32) {
    const unsigned long long rr = ready[t];
    const unsigned long long key = keep_key(d, rr);
    if (static_cast<int>(rr >> 32) <= d.small_cap && key > best) best = key;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(kFull, best, o);
    best = other > best ? other : best;
  }
  const int keep = best && allow_keep ? static_cast<int>(best & 0xffffffffu) : -1;
  // the kept column's forward offset and degree: loaded now, in flight while
  // the others are published (its raw size comes with its ready entry)
  long long kfb0 = 0, kfb1 = 0;
  if (keep >= 0 && lead) {
    kfb0 = d.fwd_ptr[keep];
    kfb1 = d.fwd_ptr[keep + 1];
  }
  int kR = 0;
  for (int base = 0; base < nready; base += 32) {
    const int t = base + lane;
    bool pub = false, big = false;
    int r = 0;
    if (t < nready) {
      const unsigned long long rr = ready[t];
      r = static_cast<int>(rr & 0xffffffffu);
      big = static_cast<int>(rr >> 32) > d.small_cap;
      pub = r != keep;
      if (r == keep) kR = static_cast<int>(rr >> 32);
    }
    publish(d, pub, big, r, lane);
  }
  if (keep < 0) return {-1, -1, 0, 0};
  kR = __reduce_max_sync(kFull, kR);
  kfb0 = __shfl_sync(kFull, kfb0, 0);
  kfb1 = __shfl_sync(kFull, kfb1, 0);
  const int kfd = static_cast<int>(kfb1 - kfb0);
  return {keep, kfd, kR - kfd, kfb0};
}

// ============================================================ big path

// The whole CTA eliminates k (R <= kBigCap, in shared memory; wider columns
// take the cooperative hub path). Returns the kept vertex (any width), -1, or
// -2. cta_prologue (the caller) has loaded fb / fdeg / R / level into sh.
__device__ __forceinline__ void cta_prologue(const FactorDev& d, int k, CtaShared& sh, bool known) {
  const int tid = threadIdx.x;
  // a kept vertex arrives with its forward offset / degree / raw size (loaded
  // by the keeper while it published the others): only a column with
  // overflow fills still needs its directory row
  if (!known || sh.R - sh.fdeg > d.c0) {
    if (tid < kDirChunks)
      sh.dirrow[tid] = static_cast<unsigned>(
          ld_relaxed(reinterpret_cast<const int*>(d.dir + static_cast<long long>(k) * kDirChunks + tid)));
  }
  if (!known && tid == 0) {
    const long long fb = d.fwd_ptr[k];
    sh.fb = fb;
    sh.fdeg = static_cast<int>(d.fwd_ptr[k + 1] - fb);
    sh.R = sh.fdeg + static_cast<int>(ld_relaxed_u64(&d.cnt[k]) >> 32);
  }
  __syncthreads();
}

// Steps 8-9 of a CTA elimination (sampling + emission, release, decrements,
// keep-one + publish) over the weight-ordered column (S.A rows, S.B weights,
// S.C suffix sums).
__device__ __forceinline__ int cta_sample_release(const FactorDev& d, int k, char* smem, CtaShared& sh,
                                                  bool allow_keep, Scratch S, int m, double lkk, int lvk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool lead = tid == 0;
  // ---- 8. sampling + emission, one sample per thread per round
  const SampleKey sk = sample_key(d, k);
  int emitted = 0;
  bool bad = false;
  for (int base = 0; base < m - 1; base += kThreads) {
    const int i = base + tid;
    int lo = 0, hi = 0, slot = 0;
    double wv = 0.0;
    const bool em = i < m - 1 && draw_sample(d, sk, k, i, m, S.A, S.B, S.C, lkk, lo, hi, wv);
    if (base == 0) SUB(3);
    if (em) {
      slot = reserve_fill_slot(d, lo);
      red_add_relaxed_u64(&d.cnt[hi], 1ull);
      bad = bad || slot < 0;
    }
    __syncwarp();
    if (em && !bad) bad = !write_fill(d, lo, slot, hi, k, wv);
    emitted += __popc(__ballot_sync(kFull, em));
  }
  if (lane == 0) sh.wcount[warp] = emitted;
  if (bad) sh.bad = 1;
  __syncthreads();
  SUB(4);
  if (sh.bad) return -2;
  if (lead) {
    int e = 0;
    for (int w2 = 0; w2 < kWarps; ++w2) e += sh.wcount[w2];
    d.samples[k] = e;
    sh.nready = 0;
    sh.bestkey = 0;
  }
  if (d.level) {  // ASAP levels, as in the warp path
    const int lk = lvk + 1;
    for (int t = tid; t < m; t += kThreads) atomicMax(&d.level[static_cast<int>(S.A[t] >> 32)], lk);
  }
  PHASE(5);
  maybe_delay(d, k, 1);

  // ---- 9. release, decrement, collect ready rows into C
  fence_acq_rel();
  __syncthreads();
  SUB(5);
  if (k == d.trace_k) snapshot_dp(d, 1, tid, kThreads);
  unsigned long long* ready = reinterpret_cast<unsigned long long*>(S.C);
  for (int t = tid; t < m; t += kThreads) {
    const unsigned long long a = S.A[t];
    const int row = static_cast<int>(a >> 32);
    const int mult = static_cast<int>(a & 0xffffffffu);
    const int fd = __ldg(&d.fdeg[row]);
    const unsigned long long old = atom_add_relaxed_u64(&d.cnt[row], static_cast<unsigned long long>(-static_cast<long long>(mult)));
    if (d.verify && dp_of(old) < mult) fail(d, kErrInternal, row);
    if (dp_of(old) == mult) {
      const unsigned long long rr = ready_info(row, fd, old);
      ready[atomicAdd(&sh.nready, 1)] = rr;
      atomicMax(&sh.bestkey, keep_key(d, rr));  // keep-one preference, decided at the barrier
    }
  }
  __syncthreads();
  const int nready = sh.nready;
  PHASE(6);
  if (k == d.trace_k) snapshot_dp(d, 2, tid, kThreads);
  maybe_delay(d, k, 2);
  if (nready == 0) return -1;

  // keep-one (any width) + publish the rest
  const unsigned long long best = sh.bestkey;
  const int keep = allow_keep ? static_cast<int>(best & 0xffffffffu) : -1;
  // the kept column's forward offset and degree: loaded now, in flight while
  // the others are published (its raw size comes with its ready entry)
  long long kfb0 = 0, kfb1 = 0;
  if (keep >= 0 && tid == kThreads - 1) {
    kfb0 = d.fwd_ptr[keep];
    kfb1 = d.fwd_ptr[keep + 1];
  }
  for (int base = 0; base < nready; base += kThreads) {
    const int t = base + tid;
    bool pub = false, big = false;
    int r = 0;
    if (t < nready) {
      const unsigned long long rr = ready[t];
      r = static_cast<int>(rr & 0xffffffffu);
      big = static_cast<int>(rr >> 32) > d.small_cap;
      pub = r != keep;
      if (r == keep) sh.next_R = static_cast<int>(rr >> 32);
    }
    publish(d, pub, big, r, lane);
  }
  __syncthreads();  // ready list (C) is reused by the next elimination; next_R visible
  if (keep >= 0 && tid == kThreads - 1) {
    sh.fb = kfb0;
    sh.fdeg = static_cast<int>(kfb1 - kfb0);
    sh.R = sh.next_R;
  }
  return keep;
}

__device__ int cta_eliminate(const FactorDev& d, int k, char* smem, CtaShared& sh, bool allow_keep) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool lead = tid == 0;
  Ctrl* ctrl = d.ctrl;
  if (d.verify && lead && dp_of(ld_relaxed_u64(&d.cnt[k])) != 0) fail(d, kErrInternal, k);
  maybe_delay(d, k, 0);

  // ---- 1. gather (counts and the directory row were fetched by cta_prologue)
  const long long fb = sh.fb;
  const int fdeg = sh.fdeg;
  // level[k] is final once k is ready; the load is first used after sampling
  const int lvk = d.level ? ld_relaxed(&d.level[k]) : 0;
  const int R = sh.R;
  const int P = next_pow2(R);
  if (lead) {
    sh.bad = 0;
    if (R > 64) atomicMax(&ctrl->max_raw, R);
  }
  __syncthreads();
  SUB(0);
  // column arena slot: the round trip overlaps the gather/sort/merge (the
  // value is first needed at the column write)
  unsigned long long start_reg = 0;
  if (lead && R > 0) start_reg = atomicAdd(&ctrl->arena_bump, static_cast<unsigned long long>(R));
  Scratch S = carve(smem, kBigCap);
  const XBuf xb{S.A, reinterpret_cast<unsigned long long*>(S.B),
                reinterpret_cast<unsigned long long*>(smem + 3 * 8 * kBigCap),
                reinterpret_cast<unsigned long long*>(smem + 4 * 8 * kBigCap)};
  int hashed = -1;  // merged column size when cta_hash_merge merged it
  {
    // gather + hash merge; the raw sort + run merge only when a row's run is
    // longer than kRunCap
    unsigned long long* stamp = d.vsub ? d.vsub + 8 * static_cast<long long>(k) + 1 : nullptr;
    const int mm = P <= kThreads       ? cta_hash_merge<1>(d, k, fb, fdeg, R, sh.dirrow, S, sh, stamp)
                   : P <= 2 * kThreads ? cta_hash_merge<2>(d, k, fb, fdeg, R, sh.dirrow, S, sh, stamp)
                                       : cta_hash_merge<4>(d, k, fb, fdeg, R, sh.dirrow, S, sh, stamp);
    if (mm >= 0) {
      hashed = mm;
      unsigned long long* ta = S.A;
      double* tb = S.B;
      S.A = S.X1;
      S.B = reinterpret_cast<double*>(S.X2);
      S.X1 = ta;
      S.X2 = reinterpret_cast<unsigned long long*>(tb);
    } else if (P <= kThreads) {
      cta_rank_raw<1>(d, k, fb, fdeg, R, sh.dirrow, S, nullptr);
    } else if (P <= 2 * kThreads) {
      cta_rank_raw<2>(d, k, fb, fdeg, R, sh.dirrow, S, nullptr);
    } else {
      cta_gather_sort_raw<4>(d, k, fb, fdeg, R, sh.dirrow, S.A, S.B, xb);
    }
  }
  discard_fills(d, k, R - fdeg, tid, kThreads);  // every gather above ended at a barrier
  PHASE(1);
  if (k == d.trace_k) snapshot_dp(d, 0, tid, kThreads);

  // ---- 3. merge runs (rows' multiplicities and left-to-right weight sums)
  int m = hashed >= 0 ? hashed : 0;
  if (lead) sh.carry_row = -1;
  __syncthreads();
  for (int base = 0; hashed < 0 && base < R; base += kThreads) {
    const int t = base + tid;
    const int row = t < R ? static_cast<int>(S.A[t] >> 32) : -2;
    const int prev = tid == 0 ? sh.carry_row : (t - 1 < R ? static_cast<int>(S.A[t - 1] >> 32) : -2);
    const bool head = t < R && row != prev;
    double acc = 0.0;
    int c = 0;
    if (head) {
      acc = S.B[t];
      c = 1;
      while (t + c < R && static_cast<int>(S.A[t + c] >> 32) == row) {
        acc = __dadd_rn(acc, S.B[t + c]);
        ++c;
      }
    }
    const unsigned b = __ballot_sync(kFull, head);
    if (lane == 0) sh.wcount[warp] = __popc(b);
    __syncthreads();  // all reads of this chunk done; counts visible
    int before = m;
    int total = 0;
#pragma unroll
    for (int w2 = 0; w2 < kWarps; ++w2) {
      before += w2 < warp ? sh.wcount[w2] : 0;
      total += sh.wcount[w2];
    }
    if (tid == kThreads - 1) sh.carry_row = row;
    if (head) {
      const int idx = before + __popc(b & lanemask_lt());
      S.A[idx] = (static_cast<unsigned long long>(static_cast<unsigned>(row)) << 32) |
                 static_cast<unsigned>(c);
      S.B[idx] = acc;
    }
    m += total;
    __syncthreads();
  }
  PHASE(2);
  if (m == 0) {
    if (lead) {
      d.diag[k] = 0.0;
      if (d.blk_done) fence_acq_rel();  // release (streamed assembly)
    }
    return -1;
  }

  // ---- 5-7. lkk + column, weight sort + suffix
  if (m >= 2 && m <= kThreads) {
    // Weight sort (broadcast all-pairs rank, one element per thread) scatters
    // the weight-ordered column to (X2, C) and leaves B (row order) intact;
    // then the two serial chains run side by side on two warps: lkk over B
    // (row order) and the suffix sums over the sorted weights (into A's
    // space). Every thread writes its column entry from registers after.
    const int g = tid;
    const unsigned long long wk = g < m ? dbits(S.B[g]) : kInfBits;
    const unsigned long long ak = g < m ? S.A[g] : ~0ull;
    unsigned long long* WA = S.X2;
    double* WB = S.C;
    double* SUF = reinterpret_cast<double*>(S.A);
    const int r = bcast_rank_cta<true>(wk, m, S.X1);
    if (g < m) {
      WA[r] = ak;
      WB[r] = bitsd(wk);
    }
    if (lead) sh.start = static_cast<long long>(start_reg);
    __syncthreads();
    SUB(2);
    if (tid == kThreads - 32) sh.lkk = serial_total(S.B, m);
    else if (lead) serial_suffix(WB, SUF, m);
    __syncthreads();
    const double lkk = sh.lkk;
    const long long start = sh.start;
    if (start + m > d.arena_cap) {
      if (lead) fail(d, kErrArena, k);
      return -2;
    }
    if (lead) {
      d.diag[k] = lkk;
      d.col_start[k] = start;
      d.col_len[k] = m;
    }
    if (g < m) {
      d.arena_rows[start + g] = static_cast<int>(ak >> 32);
      d.arena_vals[start + g] = __ddiv_rn(-bitsd(wk), lkk);
    }
    PHASE(3);
    S.C = SUF;
    S.A = WA;
    S.B = WB;
    PHASE(4);
    return cta_sample_release(d, k, smem, sh, allow_keep, S, m, lkk, lvk);
  }
  if (lead) {
    sh.lkk = serial_total(S.B, m);
    sh.start = static_cast<long long>(start_reg);
  }
  __syncthreads();
  const double lkk = sh.lkk;
  const long long start = sh.start;
  if (start + m > d.arena_cap) {
    if (lead) fail(d, kErrArena, k);
    return -2;
  }
  for (int t = tid; t < m; t += kThreads) {
    d.arena_rows[start + t] = static_cast<int>(S.A[t] >> 32);
    d.arena_vals[start + t] = __ddiv_rn(-S.B[t], lkk);
  }
  if (lead) {
    d.diag[k] = lkk;
    d.col_start[k] = start;
    d.col_len[k] = m;
  }
  PHASE(3);

  // ---- 6-7. weight sort + suffix
  if (m >= 2) {
    const int Pm = next_pow2(m);
    if (Pm <= kThreads) {
      cta_rank_weight<1>(m, S);
    } else if (Pm <= 2 * kThreads) {
      cta_rank_weight<2>(m, S);
    } else {
      cta_sort_weight_reg<4>(m, S.A, S.B, xb);
    }
    SUB(2);
    if (lead) {
      serial_suffix(S.B, S.C, m);
    }
    __syncthreads();
  }
  PHASE(4);

  return cta_sample_release(d, k, smem, sh, allow_keep, S, m, lkk, lvk);
}

// The big-CTA elimination loop: claims (or keeps) vertices and eliminates
// them in shared memory until the next one is a hub column (returns 1, vertex
// in sh.k, prologue done), a waiting CTA is asked to help a hub job (2, job
// in sh.help), or the work is over / aborted (0). Starts from sh.k (-1: claim).
template <bool HUBS>
__device__ __forceinline__ int big_loop(const FactorDev& d, char* smem, CtaShared& sh) {
  int done_local = 0;
  int k = sh.k;
  __syncthreads();  // every thread has read sh.k before thread 0 claims into it
  int chain = 0;
  int action = 0;
  while (true) {
    bool kept = true;
    if (k < 0) {
      kept = false;
      chain = 0;
      if (threadIdx.x == 0) {
        if (done_local) atomicAdd(&d.ctrl->eliminated, done_local);
        if (sh.ticket < 0) sh.ticket = atomicAdd(&d.ctrl->b_head, 1);
        int help = -1;
        const int v = claim_at(d, true, sh.ticket, HUBS ? &help : nullptr);
        sh.k = v;
        sh.help = help;
        if (v != -3) sh.ticket = -1;
      }
      done_local = 0;
      __syncthreads();
      k = sh.k;
      __syncthreads();
      if (k == -3) {  // help a posted hub phase, then wait on the same slot again
        action = 2;
        break;
      }
      if (k < 0) break;
    }
    fence_acq_rel();
    const bool lead = threadIdx.x == 0;
    PHASE(0);
    if (d.vsub && lead) {
      d.vsub[8 * static_cast<long long>(k) + 6] = (static_cast<unsigned long long>(blockIdx.x) << 8) | 0xff;
      d.vsub[8 * static_cast<long long>(k) + 7] = kept ? 1 : 2;
    }
    cta_prologue(d, k, sh, kept);
    if (sh.R > kBigCap) {  // the cooperative hub path (the caller calls it)
      if (HUBS) {
        if (lead) sh.k = k;
        action = 1;
      } else if (lead) {
        fail(d, kErrNeedHubs, k);
      }
      break;
    }
    const bool allow = ++chain < d.keep_limit;
    const int next = cta_eliminate(d, k, smem, sh, allow);
    if (next == -2) break;
    PHASE(7);
    if (d.blk_done && lead) red_add_relaxed(&d.blk_done[k >> kStreamShift], 1);  // after the release fence
    ++done_local;
    k = next;
    __syncthreads();
  }
  if (threadIdx.x == 0 && done_local) atomicAdd(&d.ctrl->eliminated, done_local);
  __syncthreads();
  return action;
}

// ============================================================ kernel
// HUBS: with the cooperative wide-column path (an ABI call into hub.cu; its
// presence alone costs the kernel registers: 132 B of spills in the CTA
// hash-merge rank loop vs none, 128^3 K3 +3%). Graphs without hub vertices
// run the instance without it; a column wider than kBigCap there aborts the
// run, which the host repeats with HUBS (capi.cu).
template <bool HUBS>
__global__ void __launch_bounds__(kThreads, 4) eliminate_kernel(const __grid_constant__ FactorDev d) {
  // the hub instance keeps its CtaShared in dynamic shared memory, where
  // hub.cu names it (k3_sh); the mesh instance keeps it static
  __shared__ CtaShared sh_static;
  CtaShared& sh = HUBS ? k3_sh() : sh_static;
  char* smem = k3_scratch();
  if (HUBS) {  // the FactorDev copy hub.cu works from
    const unsigned* src = reinterpret_cast<const unsigned*>(&d);
    unsigned* dst = reinterpret_cast<unsigned*>(k3_scratch() + kCtaSmem + kShBytes);
    for (int w = threadIdx.x; w < static_cast<int>(sizeof(FactorDev) / 4); w += kThreads) dst[w] = src[w];
    __syncthreads();
  }
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  if (ld_relaxed(&d.ctrl->status) != 0) return;

  // Role. big_layout 1: the first CTA to start on each SM is the big one, so
  // no two big CTAs share an SM (the tail's few concurrent wide columns never
  // compete for one SM's schedulers); 0: every 4th SM runs only big CTAs.
  bool big;
  if (d.big_layout == 1 && gridDim.x >= 148) {
    if (threadIdx.x == 0) {
      unsigned smid;
      asm("mov.u32 %0, %%smid;" : "=r"(smid));
      sh.k = atomicAdd(&d.ctrl->sm_slot[smid & 255], 1) == 0;
    }
    __syncthreads();
    big = sh.k != 0;
    __syncthreads();
  } else {
    big = is_big_cta();
  }
  if (!big) {
    Scratch S = carve(smem + warp * kSmallBytes, kSmallCap);
    int done_local = 0;
    Next nx{-1, -1, 0, 0};
    int chain = 0;  // consecutive kept eliminations (bounded: the FIFO queue must drain)
    while (true) {
      bool kept = true;
      if (nx.k < 0) {
        kept = false;
        chain = 0;
        int k = -1;
        if (lane == 0) {
          if (done_local) atomicAdd(&d.ctrl->eliminated, done_local);
          k = claim(d, false);
        }
        done_local = 0;
        k = __shfl_sync(kFull, k, 0);
        if (k < 0) break;
        nx = {k, -1, 0, 0};
      }
      __syncwarp();
      fence_acq_rel();  // acquire: everything published before k became ready is visible
      const int k = nx.k;
      const bool lead = lane == 0;
      PHASE(0);
      if (d.vsub && lead) {  // diagnostics: who eliminated k, and whether it was kept
        d.vsub[8 * static_cast<long long>(k) + 6] = (static_cast<unsigned long long>(blockIdx.x) << 8) | warp;
        d.vsub[8 * static_cast<long long>(k) + 7] = kept ? 1 : 2;
      }
      Next nn = warp_eliminate(d, nx, S, lane, ++chain < d.keep_limit);
      if (nn.k == -2) break;
      if (nn.k != -3) {
        PHASE(7);
        if (d.blk_done && lead) red_add_relaxed(&d.blk_done[k >> kStreamShift], 1);  // after the release fence
        ++done_local;
      }
      nx = nn.k >= 0 ? nn : Next{-1, -1, 0, 0};
    }
    if (lane == 0 && done_local) atomicAdd(&d.ctrl->eliminated, done_local);
    return;
  }

  // big CTA: the whole CTA eliminates one vertex at a time. The calls into
  // the hub path (hub.cu, an ABI call) sit outside the elimination loop with
  // the loop's state parked in shared memory, so no register is live across
  // them (values live across an ABI call cost the loop registers/spills:
  // 128^3 K3 +0.7 ms when the call sat inside the loop).
  if (threadIdx.x == 0) {
    sh.slab = -1;
    sh.slab_cap = 0;
    sh.ticket = -1;
    sh.hub_seq = 0;
    sh.k = -1;
  }
  __syncthreads();
  while (true) {
    const int action = big_loop<HUBS>(d, smem, sh);  // 0 done / abort, 1 hub column sh.k, 2 help job sh.help
    if (action == 0) break;
    if constexpr (!HUBS) {
      break;
    } else if (action == 1) {
      const int r = hub_entry(d, sh.k, -1);
      __syncthreads();
      if (r == -2) break;
      if (threadIdx.x == 0) {
        PHASE_K(7, sh.k);
        if (d.blk_done) {  // the owner acquired every chunk's stores (hub_run); release them
          fence_acq_rel();
          red_add_relaxed(&d.blk_done[sh.k >> kStreamShift], 1);
        }
        atomicAdd(&d.ctrl->eliminated, 1);
        sh.k = -1;
      }
    } else {
      hub_entry(d, -1, sh.help);
      if (threadIdx.x == 0) sh.k = -1;
    }
    __syncthreads();
  }
}

int num_sms(int device) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return sms > 0 ? sms : 148;
}

}  // namespace

template <bool HUBS>
constexpr int dyn_smem() { return HUBS ? kDynSmemHub : kCtaSmem; }

template <bool HUBS>
int occupancy_grid(int device) {
  cudaFuncSetAttribute(eliminate_kernel<HUBS>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem<HUBS>());
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, eliminate_kernel<HUBS>, kThreads, dyn_smem<HUBS>());
  if (per_sm < 1) per_sm = 1;
  return per_sm * num_sms(device);
}

// The two kernel instances live in two translation units: this one (mesh
// instance, whole-program) and eliminate_hubs.cu (the same source with
// K3_HUBS, relocatable device code so that it can call hub.cu). Relocatable
// compilation alone cost the mesh path 4% (128^3 K3 19.56 vs 20.40 ms).
int occupancy_hubs(int device);
cudaError_t launch_hubs(const FactorDev& d, int grid, cudaStream_t s);

#ifndef K3_HUBS
// The largest grid either instance launches (sizes the per-CTA hub job records)
int eliminate_occupancy_grid(int device) { return std::max(occupancy_hubs(device), occupancy_grid<false>(device)); }

cudaError_t launch_eliminate(const FactorDev& d, int grid_ctas, int reserve, cudaStream_t s, int* grid_used) {
  if (d.n == 0) return cudaSuccess;
  int dev = 0;
  cudaGetDevice(&dev);
  const int occ = d.hubs ? occupancy_hubs(dev) : occupancy_grid<false>(dev);
  int grid = grid_ctas > 0 ? grid_ctas : occ;
  // persistent: every CTA must be co-resident, beside `reserve` CTA slots
  // left to a concurrent kernel (the streamed assembly)
  if (grid > occ - reserve) grid = occ - reserve;
  if (grid < 2) grid = 2;      // at least one small and one big CTA
  if (grid_used) *grid_used = grid;
  note_launches(1);
  if (d.hubs) return launch_hubs(d, grid, s);
  eliminate_kernel<false><<<grid, kThreads, dyn_smem<false>(), s>>>(d);
  return cudaGetLastError();
}
#else
int occupancy_hubs(int device) { return occupancy_grid<true>(device); }

cudaError_t launch_hubs(const FactorDev& d, int grid, cudaStream_t s) {
  eliminate_kernel<true><<<grid, kThreads, dyn_smem<true>(), s>>>(d);
  return cudaGetLastError();
}
#endif

}  // namespace parac_gpu
