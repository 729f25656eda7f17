// K4s: the CSC assembly (ParState::assemble, proj/src/factor_par.cpp:309-345)
// streamed beside the elimination kernel instead of after it.
//
// A column of the factor is final once its position is eliminated; its place
// in the CSC output (col_ptr[k]) is final once every column before it is. On
// a random ordering the eliminations sweep the positions roughly in order:
// at 128^3, 88% of the factor's entries sit below the lowest not-yet-
// eliminated position 6 ms into the 20 ms elimination, 98% at 10 ms
// (tools/watermark.py). The streamer copies those columns while K3 still runs
// and tells the host, through per-block words in mapped pinned memory, how
// much of the output is final, so the device->host copy overlaps the elimination too.
//
// Positions are cut into blocks of kStreamBlock. K3 counts each block's
// eliminated columns (FactorDev::blk_done, one relaxed red per column after
// its release fence). A few persistent CTAs (grid taken from K3's) claim
// blocks in ascending order; for each block:
//   1. wait until all its columns are eliminated (acquire);
//   2. exclusive scan of the column lengths in shared memory;
//   3. block offsets by decoupled look-back (blk_incl[b] = the block's total,
//      then its inclusive entry offset, flagged): no serial chain per block;
//   4. col_ptr for the block, then every entry copied arena -> rows/vals,
//      a warp per group of 32 columns, lanes 32 entries apart (coalesced);
//   5. release the block to the host: system-scope fence, then its flagged
//      inclusive entry end in mapped memory (host_blk[b]); the host advances
//      over the contiguous prefix of released blocks.
// The result is bit-identical to launch_assemble's (same offsets, same
// copies). An abort of K3 (Ctrl::status != 0) ends the streamer.
#include "common.cuh"
#include "factor_kernels.cuh"

namespace parac_gpu {

void note_launches(long long k);  // defined in capi.cu

namespace {

using namespace dev;

constexpr int kStreamThreads = 256;

// exclusive scan over the CTA (red: 32 long longs); *total = the sum
__device__ __forceinline__ long long cta_exclusive_scan(long long v, long long* red, long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) red[warp] = x;
  __syncthreads();
  if (warp == 0) {
    long long t = lane < kStreamThreads / 32 ? red[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kStreamThreads / 32) red[lane] = t;
  }
  __syncthreads();
  *total = red[kStreamThreads / 32 - 1];
  const long long before = warp > 0 ? red[warp - 1] : 0;
  __syncthreads();
  return before + x - v;
}
constexpr int kPer = kStreamBlock / kStreamThreads;
constexpr unsigned long long kFlag = 1ull << 63;  // blk_incl: inclusive prefix
constexpr unsigned long long kAgg = 1ull << 62;   // blk_incl: the block's own total only
constexpr unsigned long long kVal = kAgg - 1;
constexpr int kStreamErrInternal = 17;  // Errc::internal_error

__device__ __forceinline__ void st_relaxed_u64g(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ bool aborted(const StreamDev& s) { return ld_relaxed(&s.ctrl->status) != 0; }

// Thread 0 only: wait for *p >= want. Returns false when K3 aborted. A count
// still short 10 ms after K3 has eliminated every position is a bug: it is
// reported (internal error) instead of hanging.
__device__ __forceinline__ bool wait_geq(const StreamDev& s, const int* p, int want) {
  unsigned ns = 128;
  unsigned long long over = 0;
  while (ld_relaxed(p) < want) {
    if (aborted(s)) return false;
    if (ld_relaxed(&s.ctrl->eliminated) >= s.n) {
      const unsigned long long t = globaltimer_ns();
      if (!over) over = t;
      else if (t - over > 10000000ull) {
        if (atomicCAS(&s.ctrl->status, 0, kStreamErrInternal) == 0) s.ctrl->err_info = -1 - (p - s.blk_done);
        return false;
      }
    }
    __nanosleep(ns);
    if (ns < 2048) ns <<= 1;
  }
  return true;
}

__global__ void __launch_bounds__(kStreamThreads, 4) stream_assemble_kernel(StreamDev s) {
  __shared__ long long loc[kStreamBlock + 1];
  __shared__ long long cs[kStreamBlock];  // the block's arena column starts
  __shared__ long long red[32];
  __shared__ long long base_sh;
  __shared__ int blk_sh, ok_sh;
  const int tid = threadIdx.x;
  if (tid == 0 && s.start_after > 0) {  // stay out of the wide phase's way (it is throughput-bound)
    unsigned ns = 1024;
    while (ld_relaxed(&s.ctrl->eliminated) < s.start_after && !aborted(s)) {
      __nanosleep(ns);
      if (ns < 8192) ns <<= 1;
    }
  }
  __syncthreads();
  while (true) {
    if (tid == 0) {
      const int i = atomicAdd(s.next_blk, 1);
      const int b = i < s.nb && s.claim ? s.claim[i] : i;
      blk_sh = b;
      bool ok = i < s.nb;
      if (ok) {  // every K3 counter bucket the block touches is complete
        const int a0 = s.blk_k0 ? s.blk_k0[b] : b * kStreamBlock;
        const int a1 = s.blk_k0 ? s.blk_k0[b + 1] : min(a0 + kStreamBlock, s.n);
        for (int j = a0 >> kStreamShift; ok && j <= (a1 - 1) >> kStreamShift; ++j)
          ok = wait_geq(s, &s.blk_done[j], min(kStreamBlock, s.n - j * kStreamBlock));
      }
      ok_sh = ok;
    }
    __syncthreads();
    if (!ok_sh) return;
    const int b = blk_sh;
    const int k0 = s.blk_k0 ? s.blk_k0[b] : b * kStreamBlock;
    const int cnt = (s.blk_k0 ? s.blk_k0[b + 1] : min(k0 + kStreamBlock, s.n)) - k0;
    // batch: the block's problem (rows made local to it)
    const int pid = s.pos_pid ? s.pos_pid[k0] : 0;
    const int row_base = s.pos_pid ? static_cast<int>(s.pid_base[pid]) : 0;
    fence_acq_rel();  // acquire: the block's columns (published before their counts)

    // 2. local offsets
    long long v[kPer];
    long long sum = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int c = i * kStreamThreads + tid;  // coalesced loads; offsets below need thread-contiguous runs
      if (c < cnt) cs[c] = s.col_start[k0 + c];
      v[i] = c < cnt ? s.col_len[k0 + c] : 0;
    }
    __syncthreads();  // cs holds the starts; v is reloaded thread-contiguously from shared memory below
#pragma unroll
    for (int i = 0; i < kPer; ++i) loc[i * kStreamThreads + tid] = v[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      v[i] = loc[tid * kPer + i];
      sum += v[i];
    }
    long long tot;
    long long ex = cta_exclusive_scan(sum, red, &tot);
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      loc[tid * kPer + i] = ex;
      ex += v[i];
    }
    // 3. chained prefix (block b-1 was claimed earlier by a running CTA)
    if (tid == 0) {
      loc[kStreamBlock] = tot;
      // decoupled look-back: publish this block's aggregate at once, then sum
      // predecessors' aggregates back to the first inclusive prefix
      // (batch regions: offsets are local to the member, the look-back stops
      // at the member's first block)
      const int jmin = s.blk_first ? s.blk_first[b] : 0;
      if (b > jmin) st_relaxed_u64g(&s.blk_incl[b], kAgg | static_cast<unsigned long long>(tot));
      long long bs = 0;
      bool ok = true;
      for (int j = b - 1; j >= jmin;) {
        const unsigned long long w = ld_relaxed_u64(&s.blk_incl[j]);
        if (!(w & (kFlag | kAgg))) {
          if (aborted(s)) { ok = false; break; }
          __nanosleep(32);
          continue;
        }
        bs += static_cast<long long>(w & kVal);
        if (w & kFlag) break;
        --j;
      }
      if (ok) st_relaxed_u64g(&s.blk_incl[b], kFlag | static_cast<unsigned long long>(bs + tot));
      base_sh = bs;
      ok_sh = ok;
    }
    __syncthreads();
    if (!ok_sh) return;
    const long long bs = base_sh;

    // 4. col_ptr and the entries (batch regions: the member's local col_ptr
    // at lcol[k + member], its entries from region[member])
    long long* cpo = s.lcol ? s.lcol + pid : s.col_ptr;
    for (int i = tid; i < cnt; i += kStreamThreads) cpo[k0 + i] = bs + loc[i];
    if (tid == 0) cpo[k0 + cnt] = bs + tot;  // the next block writes the same value
    long long ob = bs;  // output offset of the block's first entry
    bool fits = true;
    if (s.region) {
      ob += s.region[pid];
      fits = bs + tot <= s.reg_cap[pid];
      if (!fits && tid == 0) atomicExch(s.overflow, 1);  // the host re-assembles after K3
    }
    // Each warp copies groups of 32 consecutive columns (group g: columns
    // [32g, 32g + 32), warps take groups round robin). Lanes walk the group's
    // entries 32 apart (coalesced); an entry's column comes from a 5-step
    // search over the group's 33 offsets, not over the block's 2048 (the
    // per-entry search was the kernel's instruction bound: ncu, 10.5 cycles
    // per issue, mostly fixed-latency dependencies).
    const int warp = tid >> 5, lane = tid & 31;
    const int groups = (cnt + 31) >> 5;
    constexpr int U = 8;
    for (int g = warp; fits && g < groups; g += kStreamThreads / 32) {
      const int c0 = g << 5;
      const int nc = min(32, cnt - c0);
      const long long* gl = loc + c0;  // gl[0..nc] (loc[cnt] = tot)
      const long long g0 = gl[0], T = gl[nc] - g0;
      for (long long e0 = 0; e0 < T; e0 += 32 * U) {
        long long src[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const long long e = g0 + e0 + u * 32 + lane;
          int lo = 0;  // last column of the group with offset <= e
#pragma unroll
          for (int step = 16; step > 0; step >>= 1)
            if (lo + step < nc && gl[lo + step] <= e) lo += step;
          src[u] = cs[c0 + lo] + (e - gl[lo]);
        }
        int r[U];
        double x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (e0 + u * 32 + lane < T) {  // read once: evict-first, K3's working set keeps L2
            r[u] = __ldcs(s.arena_rows + src[u]);
            x[u] = __ldcs(s.arena_vals + src[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const long long e = e0 + u * 32 + lane;
          if (e < T) {
            __stcs(s.rows + ob + g0 + e, r[u] - row_base);
            __stcs(s.vals + ob + g0 + e, x[u]);
          }
        }
      }
    }

    // 5. release to the host: the block's inclusive entry end, flagged, in
    // mapped memory (the host finds the contiguous prefix itself)
    if (s.host_blk) {
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        __threadfence_system();
        st_sys_u64(s.host_blk + b, kFlag | static_cast<unsigned long long>(bs + tot));
      }
    }
    __syncthreads();
    const bool ok = ok_sh;
    __syncthreads();  // every thread has read ok_sh before thread 0 rewrites it
    if (!ok) return;
  }
}

}  // namespace

cudaError_t launch_stream_assemble(const StreamDev& s, int ctas, cudaStream_t st) {
  if (s.n == 0) return cudaSuccess;
  stream_assemble_kernel<<<ctas, kStreamThreads, 0, st>>>(s);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace parac_gpu
