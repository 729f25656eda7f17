// Pieces of K3 (the persistent elimination kernel) shared by its two
// translation units: eliminate.cu (the kernel, the warp and CTA paths) and
// hub.cu (the cooperative wide-column path, compiled separately so that its
// register allocation does not constrain the kernel's: see hub.cu).
#pragma once
#include "factor_device.cuh"
#include "factor_kernels.cuh"

namespace parac_gpu {
namespace k3 {

using namespace dev;
using namespace fdev;

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kEntryBytes = kSlabEntryBytes;
// small warps: A, B, C + two rank-sort segment buffers (X1, X2)
constexpr int kSmallBytes = kSmallCap * 8 * 5;
// big CTAs: A, B, C (kBigCap x 8 B each) + D, E (second exchange buffer)
constexpr int kBigBytes = kBigCap * 8 * 5;
constexpr int kCtaSmem = kWarps * kSmallBytes > kBigBytes ? kWarps * kSmallBytes : kBigBytes;

#define PHASE(i) \
  do { if (d.vtimes && lead) d.vtimes[8 * static_cast<long long>(k) + (i)] = globaltimer_ns(); } while (0)
// sub-phase stamps (record_times diagnostics): 0 setup done, 1 gather landed,
// 2 weight sort done, 3 samples drawn, 4 fills written, 5 fence done
#define PHASE_K(i, kk) \
  do { if (d.vtimes) d.vtimes[8 * static_cast<long long>(kk) + (i)] = globaltimer_ns(); } while (0)
#define SUB(i) \
  do { if (d.vsub && lead) d.vsub[8 * static_cast<long long>(k) + (i)] = globaltimer_ns(); } while (0)

// Shared state of a big CTA (one vertex at a time).
struct CtaShared {
  int k;
  int m;
  int nready;
  int emitted;
  int carry_row;
  int bad;
  double lkk;
  long long start;
  long long slab;      // this CTA's wide-column slab (entries), -1 none
  int slab_cap;
  long long fb;        // cta_prologue: forward offset, degree, raw size
  int fdeg, R;
  unsigned dirrow[kDirChunks];
  int wcount[kWarps];
  unsigned long long best[kWarps];
  int next_R;          // raw size of the kept vertex
  int mbump, mcount;   // cta_hash_merge: stage bump, distinct rows
  unsigned long long bestkey;  // keep-one: max keep_key over the rows made ready
  int hbad;            // cta_hash_merge: a run longer than kRunCap
  // cooperative wide columns (hub path)
  int ticket;          // big-queue slot this CTA waits on (-1: none), kept while it helps
  int help;            // job a waiting CTA was sent to help
  int hub_c, hub_cseq; // chunk taken, and the phase sequence it belongs to
  int hub_seq;         // owner: sequence number of its last posted phase
  HubDesc hd;          // the phase being worked on
};

// Number of keys in the sorted run A[0, len) that are < key (<= key when
// inclusive); w is the run capacity (a power of two >= len).
__device__ __forceinline__ int count_before(const unsigned long long* A, int len, int w, unsigned long long key,
                                            bool inclusive) {
  int lo = 0;
  for (int step = w >> 1; step > 0; step >>= 1) {
    const int probe = lo + step - 1;
    if (probe < len) {
      const unsigned long long m = A[probe];
      lo = (inclusive ? m <= key : m < key) ? lo + step : lo;
    }
  }
  if (lo == w - 1 && len == w) {
    const unsigned long long m = A[w - 1];
    lo += static_cast<int>(inclusive ? m <= key : m < key);
  }
  return lo;
}

// Stable sort of R <= T*ITEMS u64 keys held in registers (element g = i*T +
// tid; ties keep g order), T = 32 (one warp) or kThreads (the CTA):
//   1. rank inside the element's 32-element segment (32 broadcast loads of the
//      unsorted keys staged in X2) and write the sorted segment to X1, with
//      each key's element index alongside (IA);
//   2. merge runs pairwise, 32 -> 64 -> ... -> R: every position finds its
//      place in the merged pair with one binary search in the partner run
//      (left elements count partner keys <, right ones <=: the stable rule),
//      ping-ponging (X1, IA) <-> (X2, IB); one barrier per level.
// The dependent chain is log2(R/32) short searches instead of one search per
// other segment. Finally rank[i] = sorted position of element g.
// Raw keys (row << 32 | source+1) are unique. The weight sort needs (weight,
// row) order; its input is already row-ascending, so a STABLE sort on the
// weight bits alone gives exactly fill_sorted_view's order
// (factor_common.hpp:133-145).
template <int T, int ITEMS>
__device__ __forceinline__ void rank_sort(const unsigned long long (&k)[ITEMS], int R, unsigned long long* X1,
                                          unsigned long long* X2, int* IA, int* IB, int (&rank)[ITEMS],
                                          long long* cyc = nullptr) {
  const int tid = T == 32 ? lane_id() : static_cast<int>(threadIdx.x);
  const int lane = tid & 31;
  const int wid = tid >> 5;
  long long c0 = 0;
  if (cyc && tid == 0) c0 = clock64();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = i * T + tid;
    if (g < R) X2[g] = k[i];
  }
  if (T == 32) __syncwarp(); else __syncthreads();
  if (cyc && tid == 0) cyc[0] = clock64() - c0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int seg = i * (T / 32) + wid;
    const int len = min(32, R - seg * 32);  // <= 0: segment fully padding
    const unsigned long long* K = X2 + seg * 32;
    if (len > 0) {
      int c = 0;
#pragma unroll 8
      for (int t = 0; t < 32; ++t) {
        const unsigned long long o = t < len ? K[t] : ~0ull;
        c += static_cast<int>((o < k[i]) | ((o == k[i]) & (t < lane)));
      }
      if (lane < len) {
        X1[seg * 32 + c] = k[i];
        IA[seg * 32 + c] = seg * 32 + lane;
      }
    }
  }
  if (T == 32) __syncwarp(); else __syncthreads();
  if (cyc && tid == 0) cyc[1] = clock64() - c0;
  unsigned long long *ks = X1, *kd = X2;
  int *is = IA, *id = IB;
  for (int w = 32; w < R; w *= 2) {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int p = i * T + tid;
      if (p < R) {
        const unsigned long long key = ks[p];
        const int g = is[p];
        const int ps = p & ~(2 * w - 1);
        int np;
        if (p < ps + w) {  // left run: partner = right run, strict
          const int len = max(0, min(w, R - (ps + w)));
          np = p + count_before(ks + ps + w, len, w, key, false);
        } else {           // right run: partner = left run, inclusive
          np = (p - w) + count_before(ks + ps, w, w, key, true);
        }
        kd[np] = key;
        id[np] = g;
      }
    }
    if (T == 32) __syncwarp(); else __syncthreads();
    unsigned long long* tk = ks; ks = kd; kd = tk;
    int* ti = is; is = id; id = ti;
  }
  // ranks: the sorted position of each element index
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int p = i * T + tid;
    if (p < R) id[is[p]] = p;
  }
  if (T == 32) __syncwarp(); else __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int g = i * T + tid;
    rank[i] = g < R ? id[g] : 0;
  }
  if (cyc && tid == 0) cyc[2] = clock64() - c0;
}

// c += #{keys of pairs [q0, q1) of P below thr} (two accumulators per element)
__device__ __forceinline__ void count_below(const ulonglong2* P, int q0, int q1, unsigned long long thr, int& ca,
                                            int& cb) {
#pragma unroll 2
  for (int q = q0; q < q1; ++q) {
    const ulonglong2 p = P[q];
    ca += static_cast<int>(p.x < thr);
    cb += static_cast<int>(p.y < thr);
  }
}
// The mixed block (keys t = 2q, 2q+1 relative to the block): threshold k + 1
// before position `pos` in the block, k from it on.
__device__ __forceinline__ void count_below_mixed(const ulonglong2* P, int pairs, unsigned long long k, int pos,
                                                  int& ca, int& cb) {
  const unsigned long long k1 = k + 1;
#pragma unroll 2
  for (int q = 0; q < pairs; ++q) {
    const ulonglong2 p = P[q];
    ca += static_cast<int>(p.x < (2 * q < pos ? k1 : k));
    cb += static_cast<int>(p.y < (2 * q + 1 < pos ? k1 : k));
  }
}

// CTA: element g = threadIdx.x < R <= NT (one per thread); the first NT
// threads take part (NT < kThreads: named barrier 1, the other warps are free
// to do something else meanwhile).
template <bool STABLE, int NT = kThreads>
__device__ __forceinline__ int bcast_rank_cta(unsigned long long k, int R, unsigned long long* X) {
  const int tid = threadIdx.x, lane = tid & 31, wb = tid & ~31;
  if (tid < R) X[tid] = k;
  if (tid == 0 && (R & 1)) X[R] = ~0ull;  // pad the last pair: never below a threshold
  if (NT == kThreads) __syncthreads();
  else asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  const ulonglong2* X2 = reinterpret_cast<const ulonglong2*>(X);
  const int pairs = (R + 1) >> 1;
  int ca = 0, cb = 0;
  if (!STABLE) {
    count_below(X2, 0, pairs, k, ca, cb);
  } else {
    const int qm = min(wb >> 1, pairs), qe = min((wb + 32) >> 1, pairs);
    count_below(X2, 0, qm, k + 1, ca, cb);                   // keys before g's warp block: <= k
    count_below_mixed(X2 + qm, qe - qm, k, lane, ca, cb);    // g's warp block
    count_below(X2, qe, pairs, k, ca, cb);                   // keys after it: < k
  }
  return ca + cb;
}

// Final raw size of a vertex that just became ready, (R << 32 | row): its
// forward degree (static, loaded alongside the decrement) plus the final fill
// count returned by the decrement itself (high word of the counter).
__device__ __forceinline__ unsigned long long ready_info(int r, int fdeg, unsigned long long old_cnt) {
  return (static_cast<unsigned long long>(fdeg + static_cast<int>(old_cnt >> 32)) << 32) |
         static_cast<unsigned>(r);
}
__device__ __forceinline__ int dp_of(unsigned long long c) { return static_cast<int>(c & 0xffffffffull); }

// TestHooks::on_phase analogue (factor_par.cpp:112-120): the eliminating
// warp/CTA (t in [0, nt)) copies every dependency counter after its own
// updates of this phase are performed (the caller has fenced). Inline: an
// out-of-line call made ptxas spill around it (188 B vs 60 B in K3).
__device__ __forceinline__ void snapshot_dp(const FactorDev& d, int phase, int t, int nt) {
  long long* out = d.trace_dp + static_cast<long long>(phase) * d.n;
  for (int i = t; i < d.n; i += nt) out[i] = dp_of(ld_relaxed_u64(&d.cnt[i]));
  if (t == 0) d.trace_taken[phase] = 1;
}

// record_times diagnostics: this column's trace record and step p's 4 words
__device__ __forceinline__ unsigned long long* hub_rec(const FactorDev& d, const HubDesc& h) {
  return h.trace >= 0 ? d.hub_trace + static_cast<long long>(h.trace) * kHubTraceWords : nullptr;
}
__device__ __forceinline__ unsigned long long* hub_step(unsigned long long* rec, int p) { return rec + 8 + 4 * (p - 1); }

// dst[i] = src[i * stride], i < cnt, by threads t = 0..nt-1 (four loads in
// flight per thread: a loop of single load -> store pairs waits one L2 round
// trip per element)
template <int U = 4, typename T>
__device__ __forceinline__ void stage_in(T* dst, const T* src, int cnt, int t, int nt, int stride = 1) {
  for (int i0 = t; i0 < cnt; i0 += U * nt) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * nt;
      if (i < cnt) v[u] = __ldcg(src + static_cast<long long>(i) * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * nt < cnt) dst[i0 + u * nt] = v[u];
  }
}

// the sampling phase's id (hub.cu's phase enum), for the post from hub_chains.cu
constexpr int kHubSamplePhase = 6;

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Post phase sh.hd.phase of job `job` as sequence seq with nch chunks, first
// of them already taken (the caller keeps chunk 0 when first == 1): the
// descriptor, then the release of `next`. One full warp calls it.
__device__ __forceinline__ void hub_post_warp(const FactorDev& d, int job, CtaShared& sh, int seq, int nch,
                                              int first) {
  HubJob& J = d.hub_jobs[job];
  const int lane = threadIdx.x & 31;
  __syncwarp();
  const unsigned* src = reinterpret_cast<const unsigned*>(&sh.hd);
  unsigned* dst = reinterpret_cast<unsigned*>(&J.desc[seq & 1]);
  for (int w = lane; w < static_cast<int>(sizeof(HubDesc) / 4); w += 32) __stcg(dst + w, src[w]);
  if (lane == 0) {
    if (unsigned long long* rec = hub_rec(d, sh.hd)) {
      const int p = sh.hd.phase;
      hub_step(rec, p)[0] = globaltimer_ns();
      hub_step(rec, p)[1] = ~0ull;
    }
    st_relaxed_u64(&J.done, static_cast<unsigned long long>(seq) << 32);
  }
  fence_acq_rel();
  __syncwarp();
  if (lane == 0) {
    sh.hub_seq = seq;
    st_relaxed_u64(&J.next, (static_cast<unsigned long long>(seq) << 48) |
                                (static_cast<unsigned long long>(nch) << 24) | static_cast<unsigned>(first));
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(&d.ctrl->hub_hint), "r"(job + 1) : "memory");
  }
  __syncwarp();
}

// dst[0, cnt) = src[0, cnt) (8-byte elements, global -> shared) by the whole
// CTA with 16-byte cp.async (through L2: other SMs wrote src), all in flight
// at once and no registers held; dst and src must share their 16-byte phase.
// The caller synchronises (__syncthreads) before reading dst.
__device__ __forceinline__ void stage_async(unsigned long long* dst, const unsigned long long* src, int cnt) {
  const int tid = threadIdx.x;
  const int lead = min(cnt, (reinterpret_cast<unsigned long long>(src) & 15ull) ? 1 : 0);
  if (tid == 0 && lead) dst[0] = __ldcg(src);
  const int pairs = (cnt - lead) >> 1;
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(dst + lead));
  for (int p = tid; p < pairs; p += kThreads)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sbase + 16u * p), "l"(src + lead + 2 * p)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (tid == 0 && cnt - lead - 2 * pairs) dst[cnt - 1] = __ldcg(src + cnt - 1);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// The owner's serial chains of a hub column (hub_chains.cu): returns lkk of
// the row-ordered merged weights W[0, m); with suffix, C = suffix sums of the
// weight-ordered WB. rec: optional trace record.
// post_job >= 0: once lkk is known, warp 0 posts the sampling phase
// (pipelined: its chunks wait on HubJob::progress, which the suffix group
// publishes chunk by chunk).
__device__ double hub_chains(const double* W, const double* WB, double* C, int m, bool suffix,
                             unsigned long long* rec, int post_job);

// The hub kernel instance's dynamic shared memory: the per-CTA scratch
// (kCtaSmem bytes), then the CtaShared block. Every translation unit names it
// through this extern array, so the accesses compile to shared-memory
// instructions: a pointer handed across an out-of-line call is generic
// (LD/ST instead of LDS/STS, ~2x the latency in the serial chains).
extern __shared__ __align__(16) unsigned char k3_dyn_smem[];
// A copy of the kernel's FactorDev follows (the kernel parameter itself is
// reachable from another unit only through a generic pointer).
constexpr int kShBytes = (static_cast<int>(sizeof(CtaShared)) + 15) & ~15;
constexpr int kDevBytes = (static_cast<int>(sizeof(FactorDev)) + 15) & ~15;
constexpr int kDynSmemHub = kCtaSmem + kShBytes + kDevBytes;
__device__ __forceinline__ char* k3_scratch() { return reinterpret_cast<char*>(k3_dyn_smem); }
__device__ __forceinline__ CtaShared& k3_sh() { return *reinterpret_cast<CtaShared*>(k3_dyn_smem + kCtaSmem); }
__device__ __forceinline__ const FactorDev& k3_dev() {
  return *reinterpret_cast<const FactorDev*>(k3_dyn_smem + kCtaSmem + kShBytes);
}

// The cooperative wide-column path (hub.cu): k >= 0 -> this CTA (the owner)
// eliminates k, returns -1 or -2 (abort); k < 0 -> help job `job`.
__device__ int hub_entry(const FactorDev& d, int k, int job);

}  // namespace k3
}  // namespace parac_gpu
