// The serial FP64 chains of a hub column (lkk and the suffix sums), in their
// own translation unit: inside hub.cu they were a callee of the phase code,
// whose live registers left the chain loop too few to keep its shared-memory
// loads ahead of the adds (in-kernel 14 / 33 cycles per element for lkk /
// suffix vs 9.5 / 15 for the same code compiled alone under the same
// 64-register cap, tools/microbench/chains_iso.cu). Across units the call
// follows the ABI and this allocation is independent.
#include "k3_common.cuh"

namespace parac_gpu {
namespace k3 {

// ---- the owner's serial chains, side by side: lkk = ((0 + w0) + w1) + ...
// over the merged column in row order (factor_common.hpp:117-121), and the
// suffix sums of the weight-ordered column strictly right to left
// (sampling.hpp:72-76). Each chain is walked by one thread over
// kChainChunk-value chunks that the other warps of its group stage in shared
// memory (double-buffered, loads batched), so it runs at the FP64 add
// latency; the suffix chain's outputs go back through shared memory and its
// group writes them out coalesced. Group A (lkk): warps 0, 2, 3 (named
// barrier 1); group B (suffix): warps 1, 4..7 (named barrier 2).
constexpr int kChainChunk = 512;

__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// s + x[0] + ... + x[cnt-1], left to right; the next 8 staged values load
// while the current 8 are added
__device__ __forceinline__ double chain_sum(double s, const double* x, int cnt) {
  int t = 0;
  if (cnt >= 8) {
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = x[q];
    for (t = 8; t + 8 <= cnt; t += 8) {
      double b[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) b[q] = x[t + q];
#pragma unroll
      for (int q = 0; q < 8; ++q) s = __dadd_rn(s, a[q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = b[q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) s = __dadd_rn(s, a[q]);
  }
  for (; t < cnt; ++t) s = __dadd_rn(s, x[t]);
  return s;
}

// o[g] = x[g] + (o[g+1] or the carried s), g = cnt-1 .. 0 (first chunk: the
// chain starts at x[cnt-1] itself). Returns the carried sum. The running sum
// is the first operand (addition commutes exactly; this order is what the
// lkk chain runs at). The next 8
// values load before the current 8 are added and stored (with x and o both
// shared memory the compiler cannot move those loads above the stores
// itself), in 16-byte pairs once g is odd: one load and one store per two
// elements.
__device__ __forceinline__ double chain_suffix(double s, bool first, const double* x, double* o, int cnt) {
  int g = cnt - 1;
  if (first) {
    s = x[g];
    o[g] = s;
    --g;
  }
  if (g >= 0 && (g & 1) == 0) {  // from here g is odd: pairs (g-1, g) are 16-byte aligned
    s = __dadd_rn(s, x[g]);
    o[g] = s;
    --g;
  }
  const double2* x2 = reinterpret_cast<const double2*>(x);
  double2* o2 = reinterpret_cast<double2*>(o);
  if (g >= 7) {
    double2 a[4];  // a[q] = elements (g-1-2q, g-2q)
#pragma unroll
    for (int q = 0; q < 4; ++q) a[q] = x2[(g - 1) / 2 - q];
    for (; g - 15 >= 0; g -= 8) {
      double2 b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) b[q] = x2[(g - 9) / 2 - q];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        s = __dadd_rn(s, a[q].y);
        const double hi = s;
        s = __dadd_rn(s, a[q].x);
        o2[(g - 1) / 2 - q] = make_double2(s, hi);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) a[q] = b[q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      s = __dadd_rn(s, a[q].y);
      const double hi = s;
      s = __dadd_rn(s, a[q].x);
      o2[(g - 1) / 2 - q] = make_double2(s, hi);
    }
    g -= 8;
  }
  for (; g >= 0; --g) {
    s = __dadd_rn(s, x[g]);
    o[g] = s;
  }
  return s;
}

// Returns lkk (every thread); with suffix, C[0, m) = suffix sums of WB.
// rec: optional trace record (the ends of the two chains)
__device__ double hub_chains(const double* W, const double* WB, double* C, int m, bool suffix,
                             unsigned long long* rec, int post_job) {
  double* smem = reinterpret_cast<double*>(k3_scratch());
  constexpr int CH = kChainChunk;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = (m + CH - 1) / CH;
  double* LA = smem;           // lkk input, 2 x CH
  double* SB = smem + 2 * CH;  // suffix input, 2 x CH
  double* SO = smem + 4 * CH;  // suffix output, 2 x CH
  double* res = smem + 6 * CH;
  long long busy = 0, waitc = 0;  // trace: chain-thread cycles in the chain / at the group barrier
  if (warp == 0 || warp == 2 || warp == 3) {
    const int gt = warp == 0 ? -1 : (warp - 2) * 32 + lane;  // stager 0..63
    if (gt >= 0) stage_in<8>(LA, W, min(CH, m), gt, 64);
    named_bar(1, 96);
    double s = 0.0;
    for (int c = 0; c < nch; ++c) {
      if (gt >= 0) {
        if (c + 1 < nch) stage_in<8>(LA + ((c + 1) & 1) * CH, W + (c + 1) * CH, min(CH, m - (c + 1) * CH), gt, 64);
      } else if (lane == 0) {
        const long long c0 = clock64();
        s = chain_sum(s, LA + (c & 1) * CH, min(CH, m - c * CH));
        busy += clock64() - c0;
      }
      const long long w0 = clock64();
      named_bar(1, 96);
      waitc += clock64() - w0;
    }
    if (tid == 0) {
      res[0] = s;
      reinterpret_cast<unsigned long long*>(res)[1] = globaltimer_ns();
      reinterpret_cast<long long*>(res)[3] = busy;
      reinterpret_cast<long long*>(res)[4] = waitc;
    }
    if (post_job >= 0 && warp == 0) {  // sampling can start: lkk is known, the suffix follows
      CtaShared& sh = k3_sh();
      const FactorDev& d = k3_dev();
      if (lane == 0) {
        sh.hd.lkk = s;
        sh.hd.phase = kHubSamplePhase;
        sh.hd.pipe = 1;
      }
      hub_post_warp(d, post_job, sh, (sh.hub_seq + 1) & 0xffff, sh.hd.mt, 0);
    }
  } else if (suffix) {
    const int gt = warp == 1 ? -1 : (warp - 4) * 32 + lane;  // stager / writer 0..127
    if (gt >= 0) {
      const int lo = max(0, m - CH);
      stage_in(SB, WB + lo, m - lo, gt, 128);
    }
    named_bar(2, 160);
    double s = 0.0;
    for (int c = 0; c < nch; ++c) {
      const int lo = max(0, m - (c + 1) * CH), hi = m - c * CH;
      if (gt >= 0) {
        if (c + 1 < nch) {
          const int lo2 = max(0, m - (c + 2) * CH);
          stage_in(SB + ((c + 1) & 1) * CH, WB + lo2, lo - lo2, gt, 128);
        }
        if (c >= 1) {  // chunk c-1 = [hi, hi + CH)
          const double* o = SO + ((c - 1) & 1) * CH;
          for (int i = gt; i < CH; i += 128) __stcg(C + hi + i, o[i]);
          if (post_job >= 0) fence_acq_rel();  // release: C[hi, m) before the progress word
        }
      } else if (lane == 0) {
        const long long c0 = clock64();
        s = chain_suffix(s, c == 0, SB + (c & 1) * CH, SO + (c & 1) * CH, hi - lo);
        busy += clock64() - c0;
      }
      const long long w0 = clock64();
      named_bar(2, 160);
      waitc += clock64() - w0;
      if (post_job >= 0 && c >= 1 && gt == 0)  // sampling chunks whose suffix range is written may start
        asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(&k3_dev().hub_jobs[post_job].progress), "r"(hi)
                     : "memory");
    }
    if (gt >= 0) {  // the last chunk: [0, m - (nch - 1) * CH)
      const double* o = SO + ((nch - 1) & 1) * CH;
      for (int i = gt; i < m - (nch - 1) * CH; i += 128) __stcg(C + i, o[i]);
      if (post_job >= 0) fence_acq_rel();
    }
    if (post_job >= 0) {
      named_bar(2, 128 + 32);
      if (gt == 0)
        asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(&k3_dev().hub_jobs[post_job].progress), "r"(0)
                     : "memory");
    }
    if (tid == 32) {
      reinterpret_cast<unsigned long long*>(res)[2] = globaltimer_ns();
      reinterpret_cast<long long*>(res)[5] = busy;
      reinterpret_cast<long long*>(res)[6] = waitc;
    }
  }
  __syncthreads();
  const double lkk = res[0];
  if (rec && threadIdx.x == 0) {  // trace: the ends of the two chains
    hub_step(rec, 8)[2] = reinterpret_cast<unsigned long long*>(res)[1];
    hub_step(rec, 8)[3] = (reinterpret_cast<unsigned long long*>(res)[3] << 32) | reinterpret_cast<unsigned long long*>(res)[4];
    if (suffix) {
      hub_step(rec, 9)[2] = reinterpret_cast<unsigned long long*>(res)[2];
      hub_step(rec, 9)[3] = (reinterpret_cast<unsigned long long*>(res)[5] << 32) | reinterpret_cast<unsigned long long*>(res)[6];
    }
  }
  __syncthreads();  // res / buffers free for the caller
  return lkk;
}

}  // namespace k3
}  // namespace parac_gpu
