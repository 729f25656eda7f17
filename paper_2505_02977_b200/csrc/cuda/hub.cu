// K3's cooperative wide-column path (R-MAT hubs), see the block comment
// below. A separate translation unit, compiled with -rdc and its own
// 64-register budget: inside one unit ptxas allocates registers across calls
// (a callee gets only what its callers do not hold), so this path's code
// raised register pressure in the kernel's hot loops (measured: the CTA
// hash-merge rank loop spilled and 128^3 K3 went 19.7 -> 21.3 ms). Across
// units the call follows the ABI and the two allocations are independent.
#include "k3_common.cuh"

namespace parac_gpu {
namespace k3 {

namespace {

// ============================================================ cooperative wide columns
// Columns with more than kBigCap raw entries (R-MAT hubs: mean ~5,600 raw
// entries on the critical path at scale 20, up to ~10^5) took ~300 us on one
// SM, and they are the R-MAT critical path while most SMs idle. The owner
// (the big CTA that claimed the column) runs the elimination as phases cut
// into 256-entry chunks and posts each phase as a job (HubJob,
// factor_kernels.cuh); big CTAs waiting on the big queue take chunks
// (claim_at, via Ctrl::hub_hint) and stay with the job between its phases
// (hub_help). The owner takes chunks too, so a column completes without
// helpers. Same arithmetic and orders as the reference:
//   kHubGather  raw entries of tile c, ranked in shared memory (rank_sort;
//               raw keys are unique) -> RK/RW, each 256-entry tile sorted by
//               (row, source)
//   kHubRank    each entry's place among the other tiles (binary searches over
//               tiles staged in shared memory) -> SK/SW, the raw column sorted;
//               run heads counted per 256-entry block of the sorted order (HB)
//   kHubMerge   each run head sums its run left to right (factor_common.hpp:
//               100-113) -> merged column (row << 32 | mult, weight) in RK/RW;
//               the block's merged rows, ranked stably by weight bits, form
//               weight tile c -> WK (bits) / WB (payload) from pref[c]
//   kHubWRank   place of each weight-tile entry among the other tiles
//               (earlier tiles: ties count) -> SK (payload) / SW (weight) in
//               (weight, row) order (factor_common.hpp:133-145)
//   (owner)     lkk in row order (factor_common.hpp:117-121) and the suffix
//               sums right to left (sampling.hpp:72-76), side by side
//   kHubSample  samples i (sampling.hpp:77-83) + fill emission, the column of
//               G in row order, ASAP levels; posted from the chains as soon as
//               lkk is known, its chunks taken top down, each starting once
//               the suffix sums it searches are written (HubJob::progress)
//   kHubRelease decrements by multiplicity, ready rows published
// A phase is posted (descriptor, then the release of its `next` word) only
// after every chunk of the previous one is done, so chunks of one phase never
// read what the same phase writes (sampling reads the suffix sums only below
// the published progress).
// (kHubWTile, a separate weight-tile phase, is fused into kHubMerge; the id
// stays for the trace's step numbering)
enum : int { kHubGather = 1, kHubRank, kHubMerge, kHubWTile, kHubWRank, kHubSample, kHubRelease };
static_assert(kHubSample == kHubSamplePhase, "hub_chains.cu posts the sampling phase by number");
constexpr int kHubTile = kThreads;                    // entries per chunk, one per thread
constexpr int kHubGroup = kCtaSmem / (8 * kHubTile);  // tiles staged per shared-memory group
constexpr int kHubFullSuffix = kCtaSmem / 8;          // suffix arrays up to this size sit in shared memory

struct HubArr {
  unsigned long long *RK, *SK, *WK;
  double *RW, *SW, *WB, *C;
  int* HB;  // run heads per sorted block (in C's space: C is written after the weight rank)
};
// weight tile t (the merged rows of sorted block t) starts at pref[t] (HB's
// exclusive prefix; pref[nt] = m), right after HB in C's space
__device__ __forceinline__ int* hub_pref(const HubArr& A, int nt) { return A.HB + nt; }
__device__ __forceinline__ HubArr hub_arrays(const FactorDev& d, long long slab, int cap) {
  char* b = d.large_pool + slab * kEntryBytes;
  const long long c8 = 8ll * cap;
  return {reinterpret_cast<unsigned long long*>(b), reinterpret_cast<unsigned long long*>(b + 2 * c8),
          reinterpret_cast<unsigned long long*>(b + 4 * c8), reinterpret_cast<double*>(b + c8),
          reinterpret_cast<double*>(b + 3 * c8), reinterpret_cast<double*>(b + 5 * c8),
          reinterpret_cast<double*>(b + 6 * c8), reinterpret_cast<int*>(b + 6 * c8)};
}


// CTA sum of one int per thread (ws: kWarps ints of shared memory).
__device__ __forceinline__ int cta_sum(int v, int* ws) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) t += ws[w];
  return t;
}

// Stable rank of thread tid's key among the first cnt threads' keys (one
// 256-key tile): rank_sort's segment ranks + log2(256/32) merge passes, ~4x
// fewer shared-memory reads than the all-pairs broadcast rank (raw keys are
// unique; weight keys need the stable rule, which both give).
__device__ __forceinline__ int hub_tile_rank(unsigned long long key, int cnt, unsigned long long* X) {
  const unsigned long long k[1] = {key};
  int r[1];
  int* I = reinterpret_cast<int*>(X + 2 * kHubTile);
  rank_sort<kThreads, 1>(k, cnt, X, X + kHubTile, I, I + kHubTile, r);
  return r[0];
}

// Place of `key` (an element of sorted tile c of the sorted-tile array K[0, n))
// among the other tiles: #{keys < key} in each (STABLE: earlier tiles count
// keys <= key, the stable rule for the weight sort). Tiles are staged into
// shared memory kHubGroup at a time; four binary searches run side by side.
// PRED: pred = max(pred, largest key below `key` in the other tiles).
template <bool STABLE, bool PRED>
__device__ __forceinline__ int hub_cross_rank(const unsigned long long* K, int n, int c, unsigned long long key,
                                              bool valid, unsigned long long* X, unsigned long long& pred) {
  const int tid = threadIdx.x;
  const int nt = (n + kHubTile - 1) / kHubTile;
  int pos = 0;
  for (int g0 = 0; g0 < nt; g0 += kHubGroup) {
    const int g1 = min(nt, g0 + kHubGroup);
    const int len = min(n, g1 * kHubTile) - g0 * kHubTile;
    __syncthreads();  // the previous group (or the caller's use of X) is done
    stage_async(X, K + static_cast<long long>(g0) * kHubTile, len);
    __syncthreads();
    if (!valid) continue;
    for (int t = g0; t < g1; t += 4) {
      int lo[4], tl[4];
      unsigned long long thr[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int tt = t + q;
        lo[q] = 0;
        tl[q] = (tt < g1 && tt != c) ? min(kHubTile, n - tt * kHubTile) : 0;
        thr[q] = STABLE && tt < c ? key + 1 : key;
      }
#pragma unroll
      for (int step = kHubTile; step > 0; step >>= 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int p = lo[q] + step;
          if (p <= tl[q] && X[(t + q - g0) * kHubTile + p - 1] < thr[q]) lo[q] = p;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        pos += lo[q];
        if (PRED && lo[q] > 0) pred = max(pred, X[(t + q - g0) * kHubTile + lo[q] - 1]);
      }
    }
  }
  return pos;
}

// hub_cross_rank over tiles of variable length (<= kHubTile): tile t is
// K[toff[t], toff[t+1]). Staged kHubGroup - 1 tiles at a time (at X + the
// 16-byte phase of their first key, + their bounds after them).
template <bool STABLE>
__device__ __forceinline__ int hub_cross_rank_var(const unsigned long long* K, const int* toff_g, int nt, int c,
                                                  unsigned long long key, bool valid, unsigned long long* X) {
  constexpr int G = kHubGroup - 1;
  const int tid = threadIdx.x;
  int* tb = reinterpret_cast<int*>(X + G * kHubTile + 2);  // the group's G + 1 tile bounds
  int pos = 0;
  for (int g0 = 0; g0 < nt; g0 += G) {
    const int g1 = min(nt, g0 + G);
    __syncthreads();  // the previous group (or the caller's use of X) is done
    if (tid <= g1 - g0) tb[tid] = __ldcg(toff_g + g0 + tid);
    __syncthreads();
    const int base = tb[0], xo = base & 1;
    stage_async(X + xo, K + base, tb[g1 - g0] - base);
    __syncthreads();
    if (!valid) continue;
    for (int t = g0; t < g1; t += 4) {
      int lo[4], tl[4], st[4];
      unsigned long long thr[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int tt = t + q;
        lo[q] = 0;
        tl[q] = (tt < g1 && tt != c) ? tb[tt + 1 - g0] - tb[tt - g0] : 0;
        st[q] = tt < g1 ? xo + tb[tt - g0] - base : 0;
        thr[q] = STABLE && tt < c ? key + 1 : key;
      }
#pragma unroll
      for (int step = kHubTile; step > 0; step >>= 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int p = lo[q] + step;
          if (p <= tl[q] && X[st[q] + p - 1] < thr[q]) lo[q] = p;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) pos += lo[q];
    }
  }
  return pos;
}

// pick_by_suffix over the global suffix array through the shared-memory coarse
// index (pick_wide), fine search through L2.
__device__ __forceinline__ int hub_pick(const double* suffix, const double* coarse, int cs, int lo, int hi,
                                        double u) {
  int qlo = (lo + cs - 1) / cs, qhi = hi / cs;
  int a = lo;
  if (qlo <= qhi && coarse[qlo] > u) {
    while (qlo < qhi) {
      const int mid = qlo + (qhi - qlo + 1) / 2;
      if (coarse[mid] > u) qlo = mid; else qhi = mid - 1;
    }
    a = max(lo, qlo * cs);
  }
  int b = min(hi, a + cs);
  while (a < b) {
    const int mid = a + (b - a + 1) / 2;
    if (__ldcg(suffix + mid) > u) a = mid; else b = mid - 1;
  }
  return a;
}

__device__ __noinline__ void hub_chunk(int c, HubJob& J) {
  int* emitted = &J.emitted;
  const FactorDev& d = k3_dev();
  const HubDesc& h = k3_sh().hd;
  char* smem = k3_scratch();
  const int tid = threadIdx.x, lane = tid & 31;
  const HubArr A = hub_arrays(d, h.slab, h.cap);
  unsigned long long* X = reinterpret_cast<unsigned long long*>(smem);
  const int b0 = c * kHubTile;
  switch (h.phase) {
    case kHubGather: {
      const int cnt = min(kHubTile, h.R - b0);
      unsigned long long key = ~0ull;
      double w = 0.0;
      if (tid < cnt) load_raw_dir(d, h.k, h.fb, h.fdeg, b0 + tid, h.dirrow, key, w);
      const int r = hub_tile_rank(key, cnt, X);
      if (tid < cnt) {
        __stcg(A.RK + b0 + r, key);
        __stcg(A.RW + b0 + r, w);
      }
      if (tid == 0) __stcg(A.HB + c, 0);
      break;
    }
    case kHubRank: {
      const int cnt = min(kHubTile, h.R - b0);
      const bool v = tid < cnt;
      const unsigned long long key = v ? __ldcg(A.RK + b0 + tid) : ~0ull;
      const double w = v ? __ldcg(A.RW + b0 + tid) : 0.0;
      unsigned long long pred = v && tid > 0 ? __ldcg(A.RK + b0 + tid - 1) : 0ull;  // 0: none (rows are >= 1)
      const int pos = tid + hub_cross_rank<false, true>(A.RK, h.R, c, key, v, X, pred);
      if (v) {
        __stcg(A.SK + pos, key);
        __stcg(A.SW + pos, w);
        if ((pred >> 32) != (key >> 32)) atomicAdd(A.HB + (pos / kHubTile), 1);
      }
      break;
    }
    case kHubMerge: {
      const int cnt = min(kHubTile, h.R - b0);
      const int p = b0 + tid;
      const bool v = tid < cnt;
      const unsigned long long key = v ? __ldcg(A.SK + p) : 0ull;
      const unsigned long long prev = v && p > 0 ? __ldcg(A.SK + p - 1) : 0ull;
      const double w0 = v ? __ldcg(A.SW + p) : 0.0;
      int* ws = reinterpret_cast<int*>(X);
      int before = 0;
      for (int j = tid; j < c; j += kThreads) before += __ldcg(A.HB + j);
      before = cta_sum(before, ws);
      const bool head = v && (prev >> 32) != (key >> 32);
      const unsigned hb = __ballot_sync(kFull, head);
      __syncthreads();  // ws reused
      if (lane == 0) ws[kWarps + (tid >> 5)] = __popc(hb);
      __syncthreads();
      int off = before + __popc(hb & lanemask_lt());
#pragma unroll
      for (int w = 0; w < kWarps; ++w) off += w < (tid >> 5) ? ws[kWarps + w] : 0;
      if (head) {  // the run p, p+1, ... summed left to right, 8 loads in flight
        const unsigned row = static_cast<unsigned>(key >> 32);
        double acc = w0;
        int mult = 1;
        bool open = true;
        for (int q = p + 1; open && q < h.R; q += 8) {
          unsigned long long kk[8];
          double ww[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            kk[u] = q + u < h.R ? __ldcg(A.SK + q + u) : ~0ull;
            ww[u] = q + u < h.R ? __ldcg(A.SW + q + u) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (open && static_cast<unsigned>(kk[u] >> 32) == row) {
              acc = __dadd_rn(acc, ww[u]);
              ++mult;
            } else {
              open = false;
            }
          }
        }
        __stcg(A.RK + off, (static_cast<unsigned long long>(row) << 32) | static_cast<unsigned>(mult));
        __stcg(A.RW + off, acc);
        X[1024 + off - before] = dbits(acc);  // this block's merged rows, for its weight tile
        X[1280 + off - before] = (static_cast<unsigned long long>(row) << 32) | static_cast<unsigned>(mult);
      }
      // the weight tile of sorted block c: its merged rows (row order) ranked
      // stably by weight bits -> WK (bits) / WB (payload) at pref[c] = before
      int nh = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) nh += ws[kWarps + w];
      __syncthreads();
      const bool tv = tid < nh;
      const unsigned long long wk = tv ? X[1024 + tid] : kInfBits;
      const unsigned long long pl = tv ? X[1280 + tid] : 0ull;
      const int r = hub_tile_rank(wk, nh, X);
      if (tv) {
        __stcg(A.WK + before + r, wk);
        __stcg(reinterpret_cast<unsigned long long*>(A.WB) + before + r, pl);
      }
      if (tid == 0) __stcg(hub_pref(A, h.nt) + c, before);
      break;
    }
    case kHubWRank: {  // tile c of the weight tiles: each entry's place among the other tiles
      const int* pref = hub_pref(A, h.nt);
      const int t0 = __ldcg(pref + c), len = __ldcg(pref + c + 1) - t0;
      const bool v = tid < len;
      const unsigned long long wk = v ? __ldcg(A.WK + t0 + tid) : kInfBits;
      const unsigned long long a = v ? __ldcg(reinterpret_cast<const unsigned long long*>(A.WB) + t0 + tid) : 0ull;
      const int pos = tid + hub_cross_rank_var<true>(A.WK, pref, h.nt, c, wk, v, X);
      if (v) {
        __stcg(A.SK + pos, a);
        __stcg(A.SW + pos, bitsd(wk));
      }
      break;
    }
    case kHubSample: {
      // pipelined (h.pipe): chunks are taken top down and each waits until the
      // suffix chain has written C[b + 1, m), all its samples search
      const int m = h.m, bs = h.pipe ? (h.mt - 1 - c) * kHubTile : b0, i = bs + tid;
      const bool smp = i < m - 1, col = i < m;
      if (col) {  // the column of G (row order) and ASAP levels: lkk suffices
        const int row = static_cast<int>(__ldcg(A.RK + i) >> 32);
        d.arena_rows[h.start + i] = row;
        d.arena_vals[h.start + i] = __ddiv_rn(-__ldcg(A.RW + i), h.lkk);
        if (d.level) atomicMax(&d.level[row], h.lvk + 1);
      }
      if (h.pipe) {
        if (tid == 0) {
          int iter = 0;
          while (ld_relaxed(&J.progress) > bs + 1) {
            if ((++iter & 1023) == 0 && ld_relaxed(&d.ctrl->status) != 0) break;
            __nanosleep(64);
          }
        }
        __syncthreads();
        fence_acq_rel();  // acquire: the suffix range published by the progress word
      }
      double* S = reinterpret_cast<double*>(X);
      const bool full = m <= kHubFullSuffix;
      const int s0 = min(m, bs + 1);  // the lowest suffix entry this chunk's samples read
      if (full) {
        stage_async(reinterpret_cast<unsigned long long*>(S + s0),
                    reinterpret_cast<const unsigned long long*>(A.C + s0), m - s0);
      } else {
        const int q0 = (s0 + h.cs - 1) / h.cs;
        stage_in(S + q0, A.C + static_cast<long long>(q0) * h.cs, (m + h.cs - 1) / h.cs - q0, tid, kThreads, h.cs);
      }
      __syncthreads();
      bool em = false;
      int lo = 0, hi = 0, slot = -1;
      double wv = 0.0;
      if (smp) {  // sample_clique_sorted (sampling.hpp:77-83), as draw_sample
        const SampleKey sk = sample_key(d, h.k);
        const double s = full ? S[i + 1] : __ldcg(A.C + i + 1);
        const double u = __dmul_rn(unit_uniform(sk.seed, sk.key, static_cast<unsigned long long>(i)), s);
        const int j = full ? pick_by_suffix(S, i + 1, m - 1, u) : hub_pick(A.C, S, h.cs, i + 1, m - 1, u);
        wv = __ddiv_rn(__dmul_rn(s, __ldcg(A.SW + i)), h.lkk);
        if (wv >= kDropThreshold) {
          const int ra = static_cast<int>(__ldcg(A.SK + i) >> 32), rc = static_cast<int>(__ldcg(A.SK + j) >> 32);
          lo = min(ra, rc);
          hi = max(ra, rc);
          em = true;
        }
      }
      if (em) {
        slot = reserve_fill_slot(d, lo);
        red_add_relaxed_u64(&d.cnt[hi], 1ull);
      }
      __syncwarp();
      if (em && slot >= 0) write_fill(d, lo, slot, hi, h.k, wv);
      const int e = __popc(__ballot_sync(kFull, em));
      if (lane == 0 && e) atomicAdd(emitted, e);
      break;
    }
    case kHubRelease: {
      const int i = b0 + tid;
      bool rdy = false, big = false;
      int row = 0;
      if (i < h.m) {
        const unsigned long long a = __ldcg(A.RK + i);
        row = static_cast<int>(a >> 32);
        const int mult = static_cast<int>(a & 0xffffffffu);
        const int fd = __ldg(&d.fdeg[row]);
        const unsigned long long old =
            atom_add_relaxed_u64(&d.cnt[row], static_cast<unsigned long long>(-static_cast<long long>(mult)));
        if (d.verify && dp_of(old) < mult) fail(d, kErrInternal, row);
        if (dp_of(old) == mult) {
          rdy = true;
          big = static_cast<int>(ready_info(row, fd, old) >> 32) > d.small_cap;
        }
      }
      publish(d, rdy, big, row, lane);
      break;
    }
    default:
      break;
  }
}

// One chunk, then its completion count (release: the chunk's stores first).
__device__ __forceinline__ void hub_run_chunk(const FactorDev& d, HubJob& J, int c, char* smem, CtaShared& sh,
                                              bool own) {
  unsigned long long* rec = threadIdx.x == 0 ? hub_rec(d, sh.hd) : nullptr;
  const unsigned long long t0 = rec ? globaltimer_ns() : 0ull;
  if (rec) atomicMin(hub_step(rec, sh.hd.phase) + 1, t0);
  hub_chunk(c, J);
  fence_acq_rel();
  __syncthreads();
  if (threadIdx.x == 0) red_add_relaxed_u64(&J.done, 1ull);
  if (rec) {
    const unsigned long long t1 = globaltimer_ns();
    atomicMax(hub_step(rec, sh.hd.phase) + 2, t1);
    atomicAdd(hub_step(rec, sh.hd.phase) + 3, own ? 1ull << 32 : 1ull);
    atomicAdd(rec + 48 + sh.hd.phase, t1 - t0);
  }
}

// Helper: take chunks of job `job` (any of its phases) until it finishes, this
// CTA's own queue slot is filled, or no phase is posted for hub_linger_ns.
// The job to start with is sh.help (set by claim_at's caller).
__device__ __forceinline__ void hub_help(const FactorDev& d, char* smem, CtaShared& sh) {
  const int tid = threadIdx.x;
  unsigned long long idle0 = 0;
  if (tid == 0) idle0 = globaltimer_ns();
  while (true) {
    if (tid == 0) {
      int c = -1, seq = 0;
      int j = sh.help;
      while (true) {
        const unsigned long long nx = ld_relaxed_u64(&d.hub_jobs[j].next);
        const int nch = static_cast<int>((nx >> 24) & 0xffffffull);
        if (static_cast<int>(nx & 0xffffffull) < nch) {
          const unsigned long long old = atom_add_relaxed_u64(&d.hub_jobs[j].next, 1ull);
          if ((old & 0xffffffull) < ((old >> 24) & 0xffffffull)) {
            c = static_cast<int>(old & 0xffffffull);
            seq = static_cast<int>(old >> 48);
            break;
          }
          continue;
        }
        // no chunk left in this job's posted phase: a newer job with chunks
        // (the hint), or this job's next phase, or leave
        const int hj = ld_relaxed(&d.ctrl->hub_hint) - 1;
        if (hj >= 0 && hj != j) {
          const unsigned long long hx = ld_relaxed_u64(&d.hub_jobs[hj].next);
          if (nch == 0 || (hx & 0xffffffull) < ((hx >> 24) & 0xffffffull)) {
            j = hj;  // (this job is over: stay with the newest one)
            continue;
          }
        }
        if (nch == 0) break;  // finished, and no other job posted
        if (sh.ticket >= 0 && ld_relaxed(&d.bqueue[sh.ticket]) >= 0) break;
        if (globaltimer_ns() - idle0 > d.hub_linger_ns || ld_relaxed(&d.ctrl->status) != 0) break;
        __nanosleep(64);
      }
      sh.help = j;
      sh.hub_c = c;
      sh.hub_cseq = seq;
    }
    __syncthreads();
    const int c = sh.hub_c;
    if (c < 0) break;
    HubJob& J = d.hub_jobs[sh.help];
    fence_acq_rel();  // acquire: the phase's inputs and descriptor (published before its post)
    {
      const unsigned* src = reinterpret_cast<const unsigned*>(&J.desc[sh.hub_cseq & 1]);
      unsigned* dst = reinterpret_cast<unsigned*>(&sh.hd);
      if (tid < static_cast<int>(sizeof(HubDesc) / 4)) dst[tid] = __ldcg(src + tid);
    }
    __syncthreads();
    hub_run_chunk(d, J, c, smem, sh, false);
    if (tid == 0) idle0 = globaltimer_ns();
  }
}

// Owner: take chunks of its posted phase (first: the chunk it already holds,
// -1 none) until none is left, then wait for every chunk. Returns false when
// the factorization aborted meanwhile.
__device__ __forceinline__ bool hub_run(const FactorDev& d, int job, char* smem, CtaShared& sh, int nch, int first) {
  HubJob& J = d.hub_jobs[job];
  const int tid = threadIdx.x;
  int c = first;
  while (true) {
    if (c >= 0) hub_run_chunk(d, J, c, smem, sh, true);
    if (tid == 0) {
      const unsigned long long old = atom_add_relaxed_u64(&J.next, 1ull);
      const int cc = static_cast<int>(old & 0xffffffull);
      sh.hub_c = cc < static_cast<int>((old >> 24) & 0xffffffull) ? cc : -1;
    }
    __syncthreads();
    c = sh.hub_c;
    if (c < 0) break;
    fence_acq_rel();  // acquire: the phase's inputs
  }
  if (tid == 0) {
    const unsigned long long target = (static_cast<unsigned long long>(sh.hub_seq) << 32) |
                                      static_cast<unsigned long long>(nch);
    int iter = 0;
    sh.bad = 0;
    while (ld_relaxed_u64(&J.done) != target) {
      if ((++iter & 255) == 0 && ld_relaxed(&d.ctrl->status) != 0) {
        sh.bad = 1;
        break;
      }
      __nanosleep(32);
    }
  }
  __syncthreads();
  fence_acq_rel();  // acquire: the chunks' stores are visible
  return sh.bad == 0;
}

// Owner: post phase `phase` with nch chunks, keeping chunk 0 for itself, and run it.
__device__ __forceinline__ bool hub_phase(const FactorDev& d, int job, char* smem, CtaShared& sh, int phase, int nch) {
  __syncthreads();  // sh.hd complete
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) sh.hd.phase = phase;
    hub_post_warp(d, job, sh, (sh.hub_seq + 1) & 0xffff, nch, 1);
  }
  __syncthreads();
  return hub_run(d, job, smem, sh, nch, 0);
}

// Owner: the job is over (helpers leave: a word with no chunks and nch 0).
__device__ __forceinline__ void hub_finish(const FactorDev& d, int job, CtaShared& sh) {
  if (threadIdx.x == 0) {
    sh.hub_seq = (sh.hub_seq + 1) & 0xffff;
    st_relaxed_u64(&d.hub_jobs[job].next, static_cast<unsigned long long>(sh.hub_seq) << 48);
    atomicCAS(reinterpret_cast<int*>(&d.ctrl->hub_hint), job + 1, 0);
  }
}

// The owner's side of a cooperative wide-column elimination: the phases in
// order, with the owner's own steps between them (column size after the
// merge, the serial chains before sampling). Little state lives across the
// calls into the chunk code: out-of-line callees get the registers their
// callers do not hold (interprocedural allocation under the 64-register cap).
// Returns -1 (the rows it made ready are all published) or -2 (abort).
__device__ __forceinline__ int hub_eliminate(const FactorDev& d, int k, char* smem, CtaShared& sh) {
  const int tid = threadIdx.x;
  const bool lead = tid == 0;
  Ctrl* ctrl = d.ctrl;
  const int job = blockIdx.x;
  if (d.verify && lead && dp_of(ld_relaxed_u64(&d.cnt[k])) != 0) fail(d, kErrInternal, k);
  maybe_delay(d, k, 0);
  if (lead) {
    const int R = sh.R;
    sh.bad = 0;
    const int P = next_pow2(R);
    if (P > sh.slab_cap) {  // this CTA's slab is reused; grow it (bump allocation) when too small
      const int cap = max(P, 2 * sh.slab_cap);
      const long long base = static_cast<long long>(atomicAdd(&ctrl->large_bump, static_cast<unsigned long long>(cap)));
      if (base + cap > d.large_cap) {
        fail(d, kErrArena, k);
        sh.bad = 1;
      }
      sh.slab = base;
      sh.slab_cap = cap;
    }
    const int tix = atomicAdd(&ctrl->large_cols, 1);
    atomicMax(&ctrl->max_raw, R);
    sh.start = static_cast<long long>(atomicAdd(&ctrl->arena_bump, static_cast<unsigned long long>(R)));
    HubDesc& h = sh.hd;
    h.k = k;
    h.R = R;
    h.m = 0;
    h.nt = (R + kHubTile - 1) / kHubTile;
    h.mt = 0;
    h.fdeg = sh.fdeg;
    h.fb = sh.fb;
    h.lvk = d.level ? ld_relaxed(&d.level[k]) : 0;
    h.cs = 0;
    h.cap = sh.slab_cap;
    h.slab = sh.slab;
    h.start = 0;
    h.lkk = 0.0;
    h.trace = d.hub_trace && tix < kHubTraceCap ? tix : -1;
    if (unsigned long long* rec = hub_rec(d, h)) {
      rec[0] = static_cast<unsigned long long>(k);
      rec[1] = static_cast<unsigned long long>(R);
      rec[3] = globaltimer_ns();
    }
  }
  if (tid < kDirChunks) sh.hd.dirrow[tid] = sh.dirrow[tid];
  __syncthreads();
  if (sh.bad) return -2;
  SUB(0);
  bool ok = true;
  for (int ph = kHubGather; ok && ph <= kHubRelease; ++ph) {
    if (ph == kHubWTile) continue;  // fused into the merge (each block ranks its merged rows)
    if (ph == kHubWRank) {  // the merged column's size: run heads of every sorted block
      const HubArr A = hub_arrays(d, sh.hd.slab, sh.hd.cap);
      int m = 0;
      for (int j = tid; j < sh.hd.nt; j += kThreads) m += __ldcg(A.HB + j);
      m = cta_sum(m, reinterpret_cast<int*>(smem));
      if (lead) {
        __stcg(hub_pref(A, sh.hd.nt) + sh.hd.nt, m);  // pref[nt] = m (ordered before the post by its fence)
        sh.hd.m = m;
        sh.hd.mt = (m + kHubTile - 1) / kHubTile;
      }
      PHASE(1);
      PHASE(2);
      if (k == d.trace_k) snapshot_dp(d, 0, tid, kThreads);
      __syncthreads();
    }
    if (ph == kHubWRank && sh.hd.m < 2) continue;  // one row: nothing to sort
    bool posted = false;  // the sampling phase was posted (pipelined) from the chains
    if (ph == kHubSample) {
      PHASE(3);
      const int m = sh.hd.m;
      if (m == 0) break;  // (a raw entry always merges into a row)
      // pipelined sampling: posted as soon as lkk is known, its chunks follow
      // the suffix chain down (not with the dependency trace on this column,
      // whose snapshot sits between sampling and release)
      const bool pipe = m >= 2 && d.hub_pipe != 0 && k != d.trace_k;
      if (lead) {
        if (sh.start + m > d.arena_cap) {
          fail(d, kErrArena, k);
          sh.bad = 1;
        }
        sh.hd.start = sh.start;
        sh.hd.cs = coarse_step(m);
        sh.hd.pipe = 0;
        d.col_start[k] = sh.start;
        d.col_len[k] = m;
        d.hub_jobs[job].emitted = 0;  // ordered before the post by its fence
        d.hub_jobs[job].progress = m;
      }
      __syncthreads();
      if (sh.bad) {
        ok = false;
        break;
      }
      unsigned long long* rec = lead ? hub_rec(d, sh.hd) : nullptr;
      if (rec) {
        hub_step(rec, 8)[0] = globaltimer_ns();
        hub_step(rec, 9)[0] = hub_step(rec, 8)[0];
      }
      {
        const HubArr A = hub_arrays(d, sh.hd.slab, sh.hd.cap);
        const double lkk = hub_chains(A.RW, A.SW, A.C, m, m >= 2, rec, pipe ? job : -1);
        if (lead) {
          sh.hd.lkk = lkk;
          d.diag[k] = lkk;
        }
      }
      PHASE(4);
      __syncthreads();
      posted = pipe;
    }
    if (ph == kHubRelease) {
      PHASE(5);
      if (lead) d.samples[k] = ld_relaxed(&d.hub_jobs[job].emitted);
      maybe_delay(d, k, 1);
      if (k == d.trace_k) snapshot_dp(d, 1, tid, kThreads);
    }
    ok = posted ? hub_run(d, job, smem, sh, sh.hd.mt, -1)
                : hub_phase(d, job, smem, sh, ph, ph <= kHubMerge || ph == kHubWRank ? sh.hd.nt : sh.hd.mt);
    if (d.vsub && lead && ph <= kHubWRank) {  // wide-column stamps (tools/profile_factor.py)
      unsigned long long* wst = d.vsub + d.n * 8ll + 4ll * k;
      if (ph <= kHubMerge) wst[ph - 1] = globaltimer_ns();
      else wst[3] = globaltimer_ns();
    }
  }
  if (ok && sh.hd.m == 0 && lead) d.diag[k] = 0.0;
  PHASE(6);
  if (ok && k == d.trace_k) snapshot_dp(d, 2, tid, kThreads);
  hub_finish(d, job, sh);
  if (unsigned long long* rec = lead ? hub_rec(d, sh.hd) : nullptr) {
    rec[2] = static_cast<unsigned long long>(sh.hd.m);
    rec[4] = globaltimer_ns();
  }
  return ok ? -1 : -2;
}

}  // namespace

// The kernel's single entry into the hub path (declared in k3_common.cuh).
__device__ int hub_entry(const FactorDev&, int k, int job) {
  const FactorDev& d = k3_dev();
  char* smem = k3_scratch();
  CtaShared& sh = k3_sh();
  __syncthreads();  // every thread has read its arguments (from sh) before thread 0 rewrites sh
  if (k >= 0) return hub_eliminate(d, k, smem, sh);
  (void)job;  // == sh.help
  hub_help(d, smem, sh);
  return -1;
}

}  // namespace k3
}  // namespace parac_gpu
