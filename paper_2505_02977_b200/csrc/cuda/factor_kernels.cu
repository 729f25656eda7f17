// sm_100a kernels of the randomized approximate Cholesky factorization.
//
//   K1  pos_count_kernel / pos_fill_kernel  build_pos_graph (proj/src/factor_common.hpp:31-80)
//   K2  initial_ready_kernel                ParState ctor + publish_initial_ready
//                                           (proj/src/factor_par.cpp:144-183)
//   K3  eliminate_kernel (persistent)       one elimination per claimed queue slot:
//                                           factor_sequential's loop body
//                                           (proj/src/factor_seq.cpp:70-138) with the
//                                           par-backends' dependency hand-off
//                                           (proj/src/factor_par.cpp:282-293, 424-477)
//   K4  assemble (scan + copy)              ParState::assemble (proj/src/factor_par.cpp:309-345)
//
// Bit-exactness: every floating-point reduction is a serial
// chain in the reference's order, written with __dadd_rn/__dmul_rn/__ddiv_rn so
// no contraction can happen; sorts use unique integer keys, so any sorting
// algorithm reproduces the reference's order.
#include <atomic>
#include <cstdio>

#include "common.cuh"
#include "factor_kernels.cuh"
#include "scan.cuh"

namespace parac_gpu {

void note_launches(long long k);  // defined in capi.cu

using namespace dev;

namespace {

constexpr int kWarpsPerCta = 8;
constexpr int kThreads = kWarpsPerCta * 32;
constexpr int kRawCap = 128;  // per-warp shared-memory column capacity (entries)
// per-warp shared bytes: key0,w0,key1,w1 (8 B each), mrow,mmult (4 B), mw (8 B)
constexpr int kWarpSmemBytes = kRawCap * (8 + 8 + 8 + 8 + 4 + 4 + 8);
constexpr int kLargeEntryBytes = 48;
constexpr double kDropThreshold = 1e-300;  // factor_common.hpp:149

enum : int { kErrArena = 10, kErrStall = 11, kErrPerm = 8, kErrInternal = 17 };

__device__ __forceinline__ void fail(const FactorDev& d, int code, long long info) {
  if (atomicCAS(&d.ctrl->status, 0, code) == 0) d.ctrl->err_info = info;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void maybe_delay(const FactorDev& d, int k, int phase) {
  if (d.delay_ns > 0) {
    const unsigned long long h = mix64(static_cast<unsigned long long>(k) * 4 + phase);
    if (h % 5 == 0) __nanosleep(static_cast<unsigned>(h % static_cast<unsigned>(d.delay_ns)));
  }
}

// Views of one warp's column scratch (shared memory, or a slab of the large
// pool for columns wider than kRawCap).
struct Scratch {
  unsigned long long* key0;  // raw keys (row << 32 | source + 1), gather order
  double* w0;
  unsigned long long* key1;  // raw keys sorted
  double* w1;
  int* mrow;                 // merged, row order
  int* mmult;
  double* mw;
  // aliases, valid after the merge
  int* srow;                 // weight-sorted rows     (onto key0)
  double* sw;                // weight-sorted weights  (onto w0)
  double* suffix;            // suffix sums            (onto w1)
};

__device__ __forceinline__ Scratch carve(char* base, int cap) {
  Scratch s;
  s.key0 = reinterpret_cast<unsigned long long*>(base);
  s.w0 = reinterpret_cast<double*>(base + 8 * cap);
  s.key1 = reinterpret_cast<unsigned long long*>(base + 16 * cap);
  s.w1 = reinterpret_cast<double*>(base + 24 * cap);
  s.mw = reinterpret_cast<double*>(base + 32 * cap);
  s.mrow = reinterpret_cast<int*>(base + 40 * cap);
  s.mmult = reinterpret_cast<int*>(base + 44 * cap);
  s.srow = reinterpret_cast<int*>(s.key0);
  s.sw = s.w0;
  s.suffix = s.w1;
  return s;
}

// Address of fill slot s of position lo for READING (the chunk is known to be
// allocated: every writer finished before lo became ready).
__device__ __forceinline__ const int4* fill_slot_read(const FactorDev& d, int lo, int s) {
  if (s < d.c0) return d.pool0 + static_cast<long long>(lo) * d.c0 + s;
  const unsigned q = static_cast<unsigned>(s / d.c0) + 1u;
  const int c = 31 - __clz(q);
  const long long off = s - static_cast<long long>(d.c0) * ((1ll << c) - 1);
  const unsigned e = static_cast<unsigned>(
      ld_relaxed(reinterpret_cast<const int*>(d.dir + static_cast<long long>(lo) * kDirChunks + c - 1)));
  return d.ovf + static_cast<long long>(e - 1) * d.c0 + off;
}

// ---------------------------------------------------------------- K1
__global__ void pos_count_kernel(FactorDev d) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= d.n) return;
  const int p = d.perm[v];
  if (p < 0 || p >= d.n) {
    fail(d, kErrPerm, v);
    return;
  }
  if (atomicExch(&d.inv[p], v) != -1) fail(d, kErrPerm, v);
  int cnt = 0;
  const long long b = d.ptr[v], e = d.ptr[v + 1];
  for (long long t = b; t < e; ++t) cnt += d.perm[d.adj[t]] > p;
  d.fdeg[p] = cnt;
  d.dp[p] = static_cast<int>(e - b) - cnt;  // earlier_degree = initial dependency count
  d.fill_cnt[p] = 0;
  d.queue[p] = -1;
  d.samples[p] = 0;
}

// Warp per position: forward neighbours (q > p) in ascending position order.
__global__ void pos_fill_kernel(FactorDev d) {
  if (d.ctrl->status != 0) return;
  const int lane = lane_id();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = gw; p < d.n; p += nw) {
    const int v = d.inv[p];
    const long long b = d.ptr[v];
    const int deg = static_cast<int>(d.ptr[v + 1] - b);
    const long long out = d.fwd_ptr[p];
    if (deg <= 32) {
      int q = -1;
      double wt = 0.0;
      if (lane < deg) {
        q = __ldg(d.perm + __ldg(d.adj + b + lane));
        wt = __ldg(d.w + b + lane);
      }
      const bool keep = q > p;
      int rank = 0;
      for (int j = 0; j < deg; ++j) {
        const int qj = __shfl_sync(kFull, q, j);
        rank += (qj > p) & (qj < q);
      }
      if (keep) {
        d.fwd_to[out + rank] = q;
        d.fwd_w[out + rank] = wt;
      }
    } else {
      // Wide row: rank each kept neighbour against the whole row (L1-resident).
      for (int base = 0; base < deg; base += 32) {
        const int t = base + lane;
        int q = -1;
        double wt = 0.0;
        if (t < deg) {
          q = __ldg(d.perm + __ldg(d.adj + b + t));
          wt = __ldg(d.w + b + t);
        }
        int rank = 0;
        for (int j = 0; j < deg; ++j) {
          const int qj = __ldg(d.perm + __ldg(d.adj + b + j));
          rank += (qj > p) & (qj < q);
        }
        if (q > p) {
          d.fwd_to[out + rank] = q;
          d.fwd_w[out + rank] = wt;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- K2
__global__ void initial_ready_kernel(FactorDev d) {
  if (d.ctrl->status != 0) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ready = p < d.n && d.dp[p] == 0;
  const unsigned b = __ballot_sync(kFull, ready);
  if (b == 0) return;
  int base = 0;
  if (lane_id() == 0) base = atomicAdd(&d.ctrl->q_tail, __popc(b));
  base = __shfl_sync(kFull, base, 0);
  if (ready) d.queue[base + __popc(b & lanemask_lt())] = p;
}

// ---------------------------------------------------------------- K3
// Spin on queue slot idx (lane 0 only). Returns the vertex, or -2 on abort.
__device__ int claim(const FactorDev& d, int idx) {
  int v = ld_acquire(&d.queue[idx]);
  if (v >= 0) return v;
  unsigned long long t0 = globaltimer_ns();
  int last = ld_relaxed(&d.ctrl->q_tail);
  int iter = 0;
  while (true) {
    const int tail = ld_relaxed(&d.ctrl->q_tail);
    const int dist = idx - tail;
    unsigned ns = dist <= 0 ? 20u : (dist < 64 ? 64u * dist : 4096u);
    __nanosleep(ns);
    v = ld_acquire(&d.queue[idx]);
    if (v >= 0) return v;
    if (ld_relaxed(&d.ctrl->status) != 0) return -2;
    if ((++iter & 15) == 0) {
      const unsigned long long now = globaltimer_ns();
      if (tail != last) {
        last = tail;
        t0 = now;
      } else if (now - t0 > d.watchdog_ns) {
        fail(d, kErrStall, idx);
        return -2;
      }
    }
  }
}

// Rank-sort by a unique 64-bit key: out[rank(key)] = in. O(R^2 / 32) per warp.
__device__ __forceinline__ void rank_sort_keys(const unsigned long long* key_in, const double* w_in,
                                               int R, unsigned long long* key_out, double* w_out,
                                               int lane) {
  for (int base = 0; base < R; base += 128) {
    unsigned long long mk[4];
    double mv[4];
    int rk[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int t = base + c * 32 + lane;
      mk[c] = t < R ? key_in[t] : ~0ull;
      mv[c] = t < R ? w_in[t] : 0.0;
      rk[c] = 0;
    }
    for (int j = 0; j < R; ++j) {
      const unsigned long long kj = key_in[j];
#pragma unroll
      for (int c = 0; c < 4; ++c) rk[c] += kj < mk[c];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int t = base + c * 32 + lane;
      if (t < R) {
        key_out[rk[c]] = mk[c];
        w_out[rk[c]] = mv[c];
      }
    }
  }
}

// fill_sorted_view order (factor_common.hpp:140-144): ascending weight, ties
// by ascending row. Weights are positive, so their bit patterns order them.
__device__ __forceinline__ void rank_sort_weights(const int* mrow, const double* mw, int m,
                                                  int* srow, double* sw, int lane) {
  for (int base = 0; base < m; base += 128) {
    unsigned long long mk[4];
    int mr[4];
    int rk[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int t = base + c * 32 + lane;
      mk[c] = t < m ? static_cast<unsigned long long>(__double_as_longlong(mw[t])) : ~0ull;
      mr[c] = t < m ? mrow[t] : 0x7fffffff;
      rk[c] = 0;
    }
    for (int j = 0; j < m; ++j) {
      const unsigned long long kj = static_cast<unsigned long long>(__double_as_longlong(mw[j]));
      const int rj = mrow[j];
#pragma unroll
      for (int c = 0; c < 4; ++c) rk[c] += (kj < mk[c]) | ((kj == mk[c]) & (rj < mr[c]));
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int t = base + c * 32 + lane;
      if (t < m) {
        srow[rk[c]] = mr[c];
        sw[rk[c]] = __longlong_as_double(static_cast<long long>(mk[c]));
      }
    }
  }
}

// pick_by_suffix (include/parac/sampling.hpp:46-57)
__device__ __forceinline__ int pick_by_suffix(const double* suffix, int lo, int hi, double u) {
  while (lo < hi) {
    const int mid = lo + (hi - lo + 1) / 2;
    if (suffix[mid] > u) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// One elimination (Appendix A steps 1-9) by one warp. Returns false on abort.
__device__ bool eliminate_vertex(const FactorDev& d, int k, char* warp_smem, int lane) {
  Ctrl* ctrl = d.ctrl;
  if (d.verify && lane == 0 && ld_relaxed(&d.dp[k]) != 0) fail(d, kErrInternal, k);
  maybe_delay(d, k, 0);

  // ---- 1. gather: forward edges (source -1) ++ fills stored at k
  const long long fb = d.fwd_ptr[k];
  const int fdeg = static_cast<int>(d.fwd_ptr[k + 1] - fb);
  const int fc = ld_relaxed(&d.fill_cnt[k]);
  const int R = fdeg + fc;

  Scratch S;
  if (R <= kRawCap) {
    S = carve(warp_smem, kRawCap);
  } else {
    long long base = 0;
    if (lane == 0) {
      base = static_cast<long long>(atomicAdd(&ctrl->large_bump, static_cast<unsigned long long>(R)));
      if (base + R > d.large_cap) fail(d, kErrArena, k);
      atomicAdd(&ctrl->large_cols, 1);
      atomicMax(&ctrl->max_raw, R);
    }
    base = __shfl_sync(kFull, base, 0);
    if (base + R > d.large_cap) return false;
    S = carve(d.large_pool + base * kLargeEntryBytes, R);
  }
  if (R > 64 && R <= kRawCap && lane == 0) atomicMax(&ctrl->max_raw, R);

  for (int t = lane; t < R; t += 32) {
    int row, src1;
    double w;
    if (t < fdeg) {
      row = __ldg(d.fwd_to + fb + t);
      src1 = 0;
      w = __ldg(d.fwd_w + fb + t);
    } else {
      const int4 e = ld_cg_int4(fill_slot_read(d, k, t - fdeg));
      row = e.x;
      src1 = e.y + 1;
      w = __hiloint2double(e.w, e.z);
    }
    S.key0[t] = (static_cast<unsigned long long>(static_cast<unsigned>(row)) << 32) |
                static_cast<unsigned>(src1);
    S.w0[t] = w;
  }
  __syncwarp();

  // ---- 2. sort raw by (row, source)  (factor_common.hpp:100-104)
  rank_sort_keys(S.key0, S.w0, R, S.key1, S.w1, lane);
  __syncwarp();

  // ---- 3. merge runs: left-to-right sums, multiplicity = run length (:105-113)
  int m = 0;
  for (int base = 0; base < R; base += 32) {
    const int t = base + lane;
    bool head = false;
    int row = 0;
    if (t < R) {
      row = static_cast<int>(S.key1[t] >> 32);
      head = t == 0 || static_cast<int>(S.key1[t - 1] >> 32) != row;
    }
    const unsigned b = __ballot_sync(kFull, head);
    if (head) {
      const int idx = m + __popc(b & lanemask_lt());
      double acc = S.w1[t];
      int c = 1;
      while (t + c < R && static_cast<int>(S.key1[t + c] >> 32) == row) {
        acc = __dadd_rn(acc, S.w1[t + c]);
        ++c;
      }
      S.mrow[idx] = row;
      S.mw[idx] = acc;
      S.mmult[idx] = c;
    }
    m += __popc(b);
  }
  __syncwarp();

  if (m == 0) {  // factor_seq.cpp:92-95
    if (lane == 0) {
      d.diag[k] = 0.0;
      d.col_len[k] = 0;
      d.col_start[k] = 0;
    }
    return true;
  }

  // ---- 5. lkk = ((0 + w0) + w1) + ... in row order (factor_common.hpp:117-121)
  double lkk = 0.0;
  if (lane == 0) {
    for (int i = 0; i < m; ++i) lkk = __dadd_rn(lkk, S.mw[i]);
  }
  lkk = __shfl_sync(kFull, lkk, 0);

  // column k: rows ascending, values (-w)/lkk (factor_seq.cpp:97-102)
  long long start = 0;
  if (lane == 0) {
    start = static_cast<long long>(atomicAdd(&ctrl->arena_bump, static_cast<unsigned long long>(m)));
    if (start + m > d.arena_cap) fail(d, kErrArena, k);
  }
  start = __shfl_sync(kFull, start, 0);
  if (start + m > d.arena_cap) return false;
  for (int t = lane; t < m; t += 32) {
    d.arena_rows[start + t] = S.mrow[t];
    d.arena_vals[start + t] = __ddiv_rn(-S.mw[t], lkk);
  }
  if (lane == 0) {
    d.diag[k] = lkk;
    d.col_start[k] = start;
    d.col_len[k] = m;
  }

  // ---- 6-8. weight sort, suffix, sampling, fill emission
  int emitted = 0;
  bool bad = false;
  if (m >= 2) {
    rank_sort_weights(S.mrow, S.mw, m, S.srow, S.sw, lane);
    __syncwarp();
    if (lane == 0) {  // sampling.hpp:72-76, strictly right to left
      double s = S.sw[m - 1];
      S.suffix[m - 1] = s;
      for (int g = m - 2; g >= 0; --g) {
        s = __dadd_rn(S.sw[g], s);
        S.suffix[g] = s;
      }
    }
    __syncwarp();
    for (int base = 0; base < m - 1; base += 32) {
      const int i = base + lane;
      bool em = false;
      int lo = 0, hi = 0, slot = 0;
      double wv = 0.0;
      if (i < m - 1) {  // sampling.hpp:77-83
        const double s = S.suffix[i + 1];
        const double u = __dmul_rn(unit_uniform(d.sample_seed, k, static_cast<unsigned long long>(i)), s);
        const int j = pick_by_suffix(S.suffix, i + 1, m - 1, u);
        wv = __ddiv_rn(__dmul_rn(s, S.sw[i]), lkk);
        if (!(wv < kDropThreshold)) {
          const int a = S.srow[i], bb = S.srow[j];
          lo = min(a, bb);
          hi = max(a, bb);
          em = true;
        }
      }
      if (em) {
        slot = atomicAdd(&d.fill_cnt[lo], 1);
        red_add_relaxed(&d.dp[hi], 1);
        if (slot >= d.c0) {
          const unsigned q = static_cast<unsigned>(slot / d.c0) + 1u;
          const int c = 31 - __clz(q);
          const long long off = slot - static_cast<long long>(d.c0) * ((1ll << c) - 1);
          if (c > kDirChunks) {
            fail(d, kErrArena, lo);
            bad = true;
          } else if (off == 0) {
            const unsigned long long sz = static_cast<unsigned long long>(d.c0) << c;
            const unsigned long long at = atomicAdd(&ctrl->ovf_bump, sz);
            if (static_cast<long long>(at + sz) > d.ovf_cap) {
              fail(d, kErrArena, lo);
              bad = true;
            } else {
              st_release_u32(d.dir + static_cast<long long>(lo) * kDirChunks + c - 1,
                             static_cast<unsigned>(at / d.c0) + 1u);
            }
          }
        }
      }
      __syncwarp();
      if (em && !bad) {
        int4* dst;
        if (slot < d.c0) {
          dst = d.pool0 + static_cast<long long>(lo) * d.c0 + slot;
        } else {
          const unsigned q = static_cast<unsigned>(slot / d.c0) + 1u;
          const int c = 31 - __clz(q);
          const long long off = slot - static_cast<long long>(d.c0) * ((1ll << c) - 1);
          const unsigned* de = d.dir + static_cast<long long>(lo) * kDirChunks + c - 1;
          unsigned e = ld_acquire_u32(de);
          while (e == 0) {
            if (ld_relaxed(&ctrl->status) != 0) break;
            __nanosleep(32);
            e = ld_acquire_u32(de);
          }
          dst = e == 0 ? nullptr : d.ovf + static_cast<long long>(e - 1) * d.c0 + off;
          bad = e == 0;
        }
        if (dst) {
          const long long wb = __double_as_longlong(wv);
          st_cg_int4(dst, make_int4(hi, k, static_cast<int>(wb & 0xffffffffll),
                                    static_cast<int>(wb >> 32)));
        }
      }
      emitted += __popc(__ballot_sync(kFull, em));
    }
  }
  if (__any_sync(kFull, bad)) return false;
  if (lane == 0) d.samples[k] = emitted;
  maybe_delay(d, k, 1);

  // ---- 9. every emission visible, then decrements (factor_par.cpp:282-293)
  __threadfence();
  __syncwarp();
  for (int base = 0; base < m; base += 32) {
    const int t = base + lane;
    bool pub = false;
    int row = 0;
    if (t < m) {
      row = S.mrow[t];
      const int c = S.mmult[t];
      const int old = atom_add_acq_rel(&d.dp[row], -c);
      if (d.verify && old < c) fail(d, kErrInternal, row);
      pub = old == c;
    }
    const unsigned b = __ballot_sync(kFull, pub);
    if (b) {
      int qb = 0;
      if (lane == 0) qb = atomicAdd(&ctrl->q_tail, __popc(b));
      qb = __shfl_sync(kFull, qb, 0);
      if (pub) st_release(&d.queue[qb + __popc(b & lanemask_lt())], row);
    }
  }
  maybe_delay(d, k, 2);
  return true;
}

__global__ void __launch_bounds__(kThreads) eliminate_kernel(FactorDev d) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = lane_id();
  char* warp_smem = reinterpret_cast<char*>(smem) + (threadIdx.x >> 5) * kWarpSmemBytes;
  if (ld_relaxed(&d.ctrl->status) != 0) return;
  while (true) {
    int k = -1;
    if (lane == 0) {
      const int idx = atomicAdd(&d.ctrl->q_head, 1);
      k = idx < d.n ? claim(d, idx) : -1;
    }
    k = __shfl_sync(kFull, k, 0);
    if (k < 0) break;
    if (!eliminate_vertex(d, k, warp_smem, lane)) break;
  }
}

// ---------------------------------------------------------------- K4
__global__ void assemble_copy_kernel(FactorDev d, const long long* col_ptr, int* rows, double* vals) {
  const int lane = lane_id();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int k = gw; k < d.n; k += nw) {
    const int len = d.col_len[k];
    const long long from = d.col_start[k], to = col_ptr[k];
    for (int t = lane; t < len; t += 32) {
      rows[to + t] = d.arena_rows[from + t];
      vals[to + t] = d.arena_vals[from + t];
    }
  }
}

__global__ void sum_samples_kernel(FactorDev d) {
  long long s = 0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < d.n; p += gridDim.x * blockDim.x)
    s += d.samples[p];
  s = warp_sum(s);
  if (lane_id() == 0 && s) atomicAdd(reinterpret_cast<unsigned long long*>(&d.ctrl->total_fills),
                                     static_cast<unsigned long long>(s));
}

int g_num_sms = 0;

int num_sms(int device) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return sms > 0 ? sms : 148;
}

}  // namespace

long long scan_tiles(long long n) { return (n + kScanTile - 1) / kScanTile; }

cudaError_t launch_scan(const int* in, long long n, long long* out, long long* tile_scratch,
                        cudaStream_t s) {
  const long long tiles = scan_tiles(n);
  if (tiles == 0) return cudaMemsetAsync(out, 0, sizeof(long long), s);
  scan_tile_sums<<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, n, tile_scratch);
  scan_tile_offsets<<<1, 1024, 0, s>>>(tile_scratch, tiles);
  scan_finish<<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, n, tile_scratch, out);
  note_launches(3);
  return cudaGetLastError();
}

cudaError_t launch_pos_graph(const FactorDev& d, long long* tile_scratch, cudaStream_t s) {
  if (d.n == 0) return cudaSuccess;
  pos_count_kernel<<<(d.n + 255) / 256, 256, 0, s>>>(d);
  note_launches(1);
  cudaError_t e = launch_scan(d.fdeg, d.n, d.fwd_ptr, tile_scratch, s);
  if (e != cudaSuccess) return e;
  int dev = 0;
  cudaGetDevice(&dev);
  const int blocks = num_sms(dev) * 8;
  pos_fill_kernel<<<blocks, 256, 0, s>>>(d);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_initial_ready(const FactorDev& d, cudaStream_t s) {
  if (d.n == 0) return cudaSuccess;
  initial_ready_kernel<<<(d.n + 255) / 256, 256, 0, s>>>(d);
  note_launches(1);
  return cudaGetLastError();
}

int eliminate_occupancy_grid(int device) {
  const int smem = kWarpsPerCta * kWarpSmemBytes;
  cudaFuncSetAttribute(eliminate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, eliminate_kernel, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  return per_sm * num_sms(device);
}

cudaError_t launch_eliminate(const FactorDev& d, int grid_ctas, cudaStream_t s, int* grid_used) {
  if (d.n == 0) return cudaSuccess;
  int dev = 0;
  cudaGetDevice(&dev);
  const int smem = kWarpsPerCta * kWarpSmemBytes;
  const int occ = eliminate_occupancy_grid(dev);
  int grid = grid_ctas > 0 ? grid_ctas : occ;
  // never more warps than vertices need
  const int max_useful = (d.n + kWarpsPerCta - 1) / kWarpsPerCta;
  if (grid > max_useful) grid = max_useful;
  if (grid < 1) grid = 1;
  if (grid_used) *grid_used = grid;
  eliminate_kernel<<<grid, kThreads, smem, s>>>(d);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_assemble(const FactorDev& d, long long* col_ptr, int* rows, double* vals,
                            long long* tile_scratch, cudaStream_t s) {
  if (d.n == 0) return cudaMemsetAsync(col_ptr, 0, sizeof(long long), s);
  cudaError_t e = launch_scan(d.col_len, d.n, col_ptr, tile_scratch, s);
  if (e != cudaSuccess) return e;
  int dev = 0;
  cudaGetDevice(&dev);
  assemble_copy_kernel<<<num_sms(dev) * 8, 256, 0, s>>>(d, col_ptr, rows, vals);
  sum_samples_kernel<<<num_sms(dev) * 2, 256, 0, s>>>(d);
  note_launches(2);
  return cudaGetLastError();
}

}  // namespace parac_gpu
