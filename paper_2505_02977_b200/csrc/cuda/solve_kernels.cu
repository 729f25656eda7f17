// sm_100a kernels of the PCG solve that consumes the factor
// (proj/src/solver.cpp:32-175):
//   K5  spmv_dot_kernel          laplacian_apply (:76-93), fixed per-row order, + p.Lp partials
//   K6  sweep_forward_kernel     forward G solve (:44-52) in gather form over G's rows,
//       sweep_backward_kernel    D^+ (:54-58) fused, backward G^T solve (:60-66)
//                                Both are sync-free and persistent: warps claim positions in
//                                ASAP-level order and spin on per-position completion stamps.
//   K7  fused vector kernels     x/r update + norm, r.z, p update, mean projection
//   K8  transpose_*              G (CSC) -> G rows (CSR), k ascending per row
// The per-row triangular-solve sums run in the reference's order with
// __dmul_rn/__dsub_rn, so z = M^-1 r is bit-identical to apply_preconditioner;
// dot products use a deterministic two-level tree (run-to-run reproducible, not
// the reference's serial order), which SURVEY §8(a) a16 validated does not move
// iteration counts.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../../include/parac_gpu.h"
#include "../host/errors.hpp"
#include "common.cuh"
#include "factor_kernels.cuh"
#include "solve_kernels.cuh"

namespace parac_gpu {

void note_launches(long long k);

using namespace dev;

namespace {

constexpr int kRedBlocks = 296;  // 2 x 148 SMs: fixed => deterministic reductions
constexpr int kRedThreads = 256;
constexpr int kSweepThreads = 256;
constexpr int kRowBlock = 256;  // row entries staged per warp before the serial chain
constexpr int kFastBlock = 128;  // fast-mode batch (4 entries per lane in flight)

enum Slot { kSlotA = 0, kSlotB = 1, kSlotC = 2, kSlots = 3 };
enum Scalar { kRz0 = 0, kRz1 = 1, kPlpOk = 2, kScalars = 8 };

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Failure{internal_error, std::string(what) + ": " + cudaGetErrorString(e)};
}

template <typename T>
void dalloc(T*& p, std::size_t count) {
  if (p) cudaFree(p);
  p = nullptr;
  check(cudaMalloc(&p, std::max<std::size_t>(count, 1) * sizeof(T)), "cudaMalloc");
}
template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

int sm_count(int device) {
  int s = 0;
  cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, device);
  return s > 0 ? s : 148;
}

// ------------------------------------------------------------ reductions
__device__ __forceinline__ void block_partial(double v, double* partials) {
  __shared__ double sm[32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double s = lane < (blockDim.x >> 5) ? sm[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) partials[blockIdx.x] = s;
  }
}

// Sum of kRedBlocks partials in a fixed order (every reader gets the same bits).
__device__ __forceinline__ double sum_partials(const double* partials) {
  double s = 0.0;
  for (int i = 0; i < kRedBlocks; ++i) s += partials[i];
  return s;
}

__device__ __forceinline__ double block_scalar(const double* partials) {
  __shared__ double v;
  if (threadIdx.x == 0) v = sum_partials(partials);
  __syncthreads();
  return v;
}

// -------------------------------------------------------------- graph prep
// wdeg: left-to-right sum in ascending-neighbour order (src/graph.cpp:66-75)
__global__ void wdeg_kernel(int n, const long long* ptr, const double* w, double* wdeg) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  double s = 0.0;
  for (long long t = ptr[v]; t < ptr[v + 1]; ++t) s = __dadd_rn(s, w[t]);
  wdeg[v] = s;
}

__device__ int cc_find(int* parent, int v) {
  int p = parent[v];
  while (p != v) {
    const int g = parent[p];
    if (g != p) parent[v] = g;  // path halving (benign race)
    v = p;
    p = g;
  }
  return v;
}

__global__ void cc_init(int n, int* parent) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) parent[v] = v;
}

// Union-find hooking over every edge (u < v): link the larger root under the smaller.
__global__ void cc_hook(int n, const long long* ptr, const int* adj, int* parent) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  for (long long t = ptr[v]; t < ptr[v + 1]; ++t) {
    const int u = adj[t];
    if (u <= v) continue;
    while (true) {
      int ru = cc_find(parent, u), rv = cc_find(parent, v);
      if (ru == rv) break;
      const int hi = max(ru, rv), lo = min(ru, rv);
      if (atomicCAS(&parent[hi], hi, lo) == hi) break;
    }
  }
}

__global__ void cc_count_roots(int n, int* parent, int* count) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  int root = 0;
  if (v < n) root = cc_find(parent, v) == v;
  root = warp_sum(root);
  if ((threadIdx.x & 31) == 0 && root) atomicAdd(count, root);
}

// ------------------------------------------------------------- factor prep
__global__ void inverse_perm_kernel(int n, const int* perm, int* inv) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) inv[perm[v]] = v;
}

__global__ void gt_count_kernel(long long nnz, const int* rows, int* cnt) {
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < nnz;
       t += static_cast<long long>(gridDim.x) * blockDim.x)
    atomicAdd(&cnt[rows[t]], 1);
}

// Warp per column k: scatter (k, G(r,k)) into row r (unordered within a row).
__global__ void gt_fill_kernel(int n, const long long* col_ptr, const int* rows,
                               const double* vals, const long long* gt_ptr, int* cursor,
                               int* gt_col, double* gt_val) {
  const int lane = lane_id();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int k = gw; k < n; k += nw) {
    for (long long t = col_ptr[k] + lane; t < col_ptr[k + 1]; t += 32) {
      const int r = rows[t];
      const long long at = gt_ptr[r] + atomicAdd(&cursor[r], 1);
      gt_col[at] = k;
      gt_val[at] = vals[t];
    }
  }
}

// Warp per row: sort the row's (k, value) by k (unique) by ranking.
__global__ void gt_sort_kernel(int n, const long long* gt_ptr, int* gt_col, double* gt_val) {
  const int lane = lane_id();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = gw; r < n; r += nw) {
    const long long b = gt_ptr[r];
    const int len = static_cast<int>(gt_ptr[r + 1] - b);
    if (len <= 1) continue;
    if (len <= 32) {
      int k = lane < len ? gt_col[b + lane] : 0x7fffffff;
      double v = lane < len ? gt_val[b + lane] : 0.0;
      int rank = 0;
      for (int j = 0; j < len; ++j) rank += __shfl_sync(kFull, k, j) < k;
      __syncwarp();
      if (lane < len) {
        gt_col[b + rank] = k;
        gt_val[b + rank] = v;
      }
    } else {
      // In-place odd-even transposition is O(len^2); rows this long are rare.
      for (int phase = 0; phase < len; ++phase) {
        for (int i = 2 * lane + (phase & 1); i + 1 < len; i += 64) {
          const int a = gt_col[b + i], c = gt_col[b + i + 1];
          if (a > c) {
            gt_col[b + i] = c;
            gt_col[b + i + 1] = a;
            const double va = gt_val[b + i];
            gt_val[b + i] = gt_val[b + i + 1];
            gt_val[b + i + 1] = va;
          }
        }
        __syncwarp();
      }
    }
  }
}

// Relaxed polling with exponential backoff (no L1 invalidation per poll); the
// caller follows with fence_acq_rel() before reading the producer's data.
__device__ __forceinline__ void wait_stamp(const int* flag, int stamp) {
  if (ld_relaxed(flag) >= stamp) return;
  unsigned ns = 32;
  do {
    __nanosleep(ns);
    if (ns < 512) ns <<= 1;
  } while (ld_relaxed(flag) < stamp);
}

// ASAP levels of the factor DAG (schedule_levels, src/factor_par.cpp:659-684):
// level[r] = 1 + max level over G's row r. Sync-free, positions claimed in
// ascending order (all dependencies are earlier positions => deadlock-free).
__global__ void level_kernel(int n, const long long* gt_ptr, const int* gt_col, int* level,
                             int* flags, int stamp, int* counter) {
  const int lane = lane_id();
  while (true) {
    int r = 0;
    if (lane == 0) r = atomicAdd(counter, 1);
    r = __shfl_sync(kFull, r, 0);
    if (r >= n) return;
    int lv = 0;
    for (long long t = gt_ptr[r] + lane; t < gt_ptr[r + 1]; t += 32) {
      const int k = gt_col[t];
      wait_stamp(&flags[k], stamp);
      fence_acq_rel();
      lv = max(lv, ld_relaxed(&level[k]));
    }
    lv = warp_max(lv) + 1;
    if (lane == 0) {
      level[r] = lv;
      st_release(&flags[r], stamp);
    }
  }
}

__global__ void level_hist_kernel(int n, const int* level, int* hist, int* depth) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  atomicAdd(&hist[level[r]], 1);
  atomicMax(depth, level[r]);
}

__global__ void level_scatter_kernel(int n, const int* level, const long long* off, int* cursor,
                                     int* order) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int l = level[r];
  order[off[l] + atomicAdd(&cursor[l], 1)] = r;
}

// ---------------------------------------------------------------- K5 / K7
// lp = L p (laplacian_apply order) and partial p.lp.
__global__ void spmv_dot_kernel(int n, const long long* ptr, const int* adj, const double* w,
                                const double* wdeg, const double* p, double* lp,
                                double* partials) {
  double acc_dot = 0.0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    double acc = __dmul_rn(wdeg[v], p[v]);
    for (long long t = ptr[v]; t < ptr[v + 1]; ++t) acc = __dsub_rn(acc, __dmul_rn(w[t], p[adj[t]]));
    lp[v] = acc;
    acc_dot += p[v] * acc;
  }
  block_partial(acc_dot, partials);
}

// partial sum and sum of squares helpers
__global__ void sum_kernel(int n, const double* a, double* partials) {
  double s = 0.0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) s += a[v];
  block_partial(s, partials);
}

// out = a - mean(a) (mean from partials), plus partial ||out||^2. Optionally
// also r = out and x = 0 (PCG start, solver.cpp:107-119).
__global__ void center_kernel(int n, const double* a, const double* sum_partials_in, double* out,
                              double* r, double* x, double* partials) {
  __shared__ double mean;
  if (threadIdx.x == 0) mean = sum_partials(sum_partials_in) / static_cast<double>(n);
  __syncthreads();
  double s = 0.0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const double o = a[v] - mean;
    out[v] = o;
    if (r) r[v] = o;
    if (x) x[v] = 0.0;
    s += o * o;
  }
  block_partial(s, partials);
}

// alpha = rz / p.lp; x += alpha p; r -= alpha lp; partial ||r||^2 (solver.cpp:133-140).
// If p.lp <= 0 nothing is updated and the flag is raised (solver.cpp:134).
__global__ void update_xr_kernel(int n, const double* plp_partials, const double* scalars_in,
                                 int rz_slot, double* x, double* r, const double* p,
                                 const double* lp, double* partials, double* flag_out) {
  __shared__ double alpha;
  __shared__ int ok;
  if (threadIdx.x == 0) {
    const double plp = sum_partials(plp_partials);
    ok = plp > 0.0;
    alpha = ok ? scalars_in[rz_slot] / plp : 0.0;
    if (blockIdx.x == 0) *flag_out = ok ? 1.0 : 0.0;
  }
  __syncthreads();
  double s = 0.0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    double rv = r[v];
    if (ok) {
      x[v] += alpha * p[v];
      rv -= alpha * lp[v];
      r[v] = rv;
    }
    s += rv * rv;
  }
  block_partial(s, partials);
}

// z (label space) = zb[perm[v]]; partial r.z (solver.cpp:145-146 / :122-124).
__global__ void gather_z_dot_kernel(int n, const int* perm, const double* zb, const double* r,
                                    double* z, double* partials) {
  double s = 0.0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const double zv = zb[perm[v]];
    z[v] = zv;
    s += r[v] * zv;
  }
  block_partial(s, partials);
}

// beta = rz_next / rz; p = z + beta p (solver.cpp:146-152). first: p = z.
__global__ void update_p_kernel(int n, const double* rz_partials, double* scalars, int rz_old,
                                int rz_new, int first, const double* z, double* p) {
  __shared__ double beta;
  if (threadIdx.x == 0) {
    const double rzn = sum_partials(rz_partials);
    beta = first ? 0.0 : rzn / scalars[rz_old];
    if (blockIdx.x == 0) scalars[rz_new] = rzn;
  }
  __syncthreads();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    p[v] = first ? z[v] : z[v] + beta * p[v];
}

__global__ void copy_kernel(int n, const double* a, double* b) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) b[v] = a[v];
}

// partial ||a - b||^2
__global__ void diff_norm_kernel(int n, const double* a, const double* b, double* partials) {
  double s = 0.0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const double d = a[v] - b[v];
    s += d * d;
  }
  block_partial(s, partials);
}

// ------------------------------------------------------------------- K6
// Level-pipelined triangular sweeps. Rows are claimed in ASAP-level order
// (forward: ascending, backward: descending). A row of level L starts once
// every row of level L-1 (forward) / L+1 (backward) has finished: by
// induction all its dependencies are then complete, so only one counter is
// polled per row (lane 0, backoff by distance to the highest finished level)
// instead of one flag per dependency -- per-dependency polling by ~9.5k warps
// saturated L2 with requests. done[L] counts finished rows of level L; the
// finishing row's increment follows a release fence, the waiter's relaxed
// read is followed by an acquire fence.
__device__ __forceinline__ int level_size(const long long* lvl_off, int L) {
  return static_cast<int>(lvl_off[L + 1] - lvl_off[L]);
}

// Wait until level L is complete. The sleep follows the distance to the
// finishing front, probed on level-specific counters 1, 3 and 15 levels back
// in sweep order (step = -1 forward, +1 backward): no word is polled by every
// waiter, and the thousands of waiters far from the front poll rarely, which
// keeps L2 latency low for the rows on the critical path.
__device__ __forceinline__ bool level_done(const int* done, const long long* lvl_off, int L, int lo,
                                           int hi) {
  return L < lo || L > hi || ld_relaxed(&done[L]) >= level_size(lvl_off, L);
}

__device__ __forceinline__ void wait_level(const int* done, const long long* lvl_off, int L, int step,
                                           int depth) {
  const int target = level_size(lvl_off, L);
  if (ld_relaxed(&done[L]) >= target) return;
  // Near the front every waiter of the next level polls done[L]; a wide next
  // level means many pollers of one word, so the near interval grows with it.
  const int nxt = L - step;
  const int pollers = (nxt >= 1 && nxt <= depth) ? level_size(lvl_off, nxt) : 1;
  const unsigned near_ns = 32u + static_cast<unsigned>(min(pollers, 4096)) / 4u;
  // The distance probes cost dependent round trips: re-classify only every 8th
  // poll, so a waiter near the front re-checks done[L] every ~near_ns + 1 RT.
  unsigned ns = near_ns;
  const unsigned long long t0 = globaltimer_ns();
  for (int it = 0;; ++it) {
    if ((it & 7) == 0 || ns >= 1024) {  // long sleepers re-probe every time
      // done[0] (level 0 does not exist) is the sweep's abort word: a wait
      // that exceeds 20 s raises it, and every waiter then bails out.
      if (ld_relaxed(&done[0]) != 0) return;
      if (globaltimer_ns() - t0 > 20000000000ull) {
        atomicExch(const_cast<int*>(&done[0]), 1);
        return;
      }
      // sleep ~ distance to the front (levels take ~3-30 us each): a waiter
      // far ahead must not poll -- thousands of early waiters polling slowed
      // the L2 for the rows on the critical path by 2-3x (measured).
      if (level_done(done, lvl_off, L + step, 1, depth)) ns = near_ns;
      else if (level_done(done, lvl_off, L + 2 * step, 1, depth)) ns = 1024;
      else if (level_done(done, lvl_off, L + 4 * step, 1, depth)) ns = 3072;
      else if (level_done(done, lvl_off, L + 8 * step, 1, depth)) ns = 8192;
      else if (level_done(done, lvl_off, L + 16 * step, 1, depth)) ns = 16384;
      else ns = 32768;
    }
    __nanosleep(ns);
    if (ld_relaxed(&done[L]) >= target) return;
  }
}

__device__ __forceinline__ void finish_row(int* done, int L) {
  fence_acq_rel();  // release: this row's value before the count
  atomicAdd(&done[L], 1);
}

// acc -= prod[0] - ... - prod[cnt-1], strictly in order, by lane 0 from the
// warp's shared slots (loads hoisted 4 at a time; ~one DSUB latency per term).
__device__ __forceinline__ double serial_sub(double acc, const double* buf, int cnt) {
  int j = 0;
  for (; j + 8 <= cnt; j += 8) {
    double p[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) p[q] = buf[j + q];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = __dsub_rn(acc, p[q]);
  }
  for (; j < cnt; ++j) acc = __dsub_rn(acc, buf[j]);
  return acc;
}

// Row j of the level order belongs to warp j mod W: a level's rows are spread
// round-robin and consecutive narrow levels land on consecutive warps, so the
// warp owning a tail row arrives there early and stages it while waiting.
__device__ __forceinline__ long long first_row(long long lb, int w, int W) {
  return lb + ((w - lb % W) % W + W) % W;
}

// Products G(.,.) * x[idx] of one block of a row into the warp's shared slots.
// All index loads, then all value loads, then the stores: explicit register
// staging, because global loads through generic pointers are otherwise not
// hoisted above the shared-memory stores (measured 50 -> ~12 cycles/entry).
// skip_zero replaces terms with x == 0 by +0.0 (see the forward sweep).
__device__ __forceinline__ void stage_products(const int* idx, const double* g, const double* x, int cnt,
                                               int lane, bool skip_zero, double* wbuf) {
  constexpr int Q = kRowBlock / 32;
  int ci[Q];
  double xv[Q], gv[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) ci[q] = q * 32 + lane < cnt ? idx[q * 32 + lane] : 0;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    xv[q] = q * 32 + lane < cnt ? __ldcg(x + ci[q]) : 0.0;
    gv[q] = q * 32 + lane < cnt ? g[q * 32 + lane] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < Q; ++q)
    if (q * 32 + lane < cnt) wbuf[q * 32 + lane] = (skip_zero && xv[q] == 0.0) ? 0.0 : __dmul_rn(gv[q], xv[q]);
}

// Wide levels (>= kLaneRowsPerWarp rows per warp): one row per LANE, summed
// sequentially in the reference's order (so these rows are bit-exact in both
// modes) -- 32 independent rows per warp instead of one keeps the first,
// widest levels (10^5 rows each at 128^3) from being latency-bound per row.
constexpr int kLaneRowsPerWarp = 2;

__device__ __forceinline__ bool lane_mode(const long long* lvl_off, int L, int W) {
  return level_size(lvl_off, L) >= kLaneRowsPerWarp * W;
}

// Forward rows of level L, one per lane (gather form, k ascending, zero skip).
__device__ __forceinline__ void lane_level_forward(int L, int depth, int w, int W, int lane,
                                                   const int* order, const long long* lvl_off,
                                                   const long long* gt_ptr, const int* gt_col,
                                                   const double* gt_val, const double* diag,
                                                   const int* inv, const double* rvec, double* yf,
                                                   double* yd, int* done) {
  const long long lb = lvl_off[L], le = lvl_off[L + 1];
  const long long ntask = (le - lb + 31) / 32;
  bool waited = L == 1;
  for (long long t = w; t < ntask; t += W) {
    if (!waited) {
      if (lane == 0) wait_level(done, lvl_off, L - 1, -1, depth);
      __syncwarp();
      fence_acq_rel();
      waited = true;
    }
    const long long j = lb + t * 32 + lane;
    if (j < le) {
      const int r = order[j];
      double acc = rvec[inv[r]];
      const long long b = gt_ptr[r], e = gt_ptr[r + 1];
      for (long long q = b; q < e; ++q) {
        const double yk = __ldcg(yf + gt_col[q]);
        if (yk != 0.0) acc = __dsub_rn(acc, __dmul_rn(gt_val[q], yk));
      }
      yf[r] = acc;
      const double dd = diag[r];
      yd[r] = dd > 0.0 ? __ddiv_rn(acc, dd) : 0.0;
    }
    const unsigned ok = __ballot_sync(kFull, j < le);
    fence_acq_rel();
    __syncwarp();
    if (lane == 0) atomicAdd(&done[L], __popc(ok));
  }
}

// Backward rows (columns of G) of level L, one per lane, rows ascending.
__device__ __forceinline__ void lane_level_backward(int L, int depth, int w, int W, int lane,
                                                    const int* order, const long long* lvl_off,
                                                    const long long* col_ptr, const int* rows,
                                                    const double* vals, const double* yd, double* zb,
                                                    int* done) {
  const long long lb = lvl_off[L], le = lvl_off[L + 1];
  const long long ntask = (le - lb + 31) / 32;
  bool waited = L == depth;
  for (long long t = w; t < ntask; t += W) {
    if (!waited) {
      if (lane == 0) wait_level(done, lvl_off, L + 1, +1, depth);
      __syncwarp();
      fence_acq_rel();
      waited = true;
    }
    const long long j = lb + t * 32 + lane;
    if (j < le) {
      const int k = order[j];
      double acc = yd[k];
      const long long b = col_ptr[k], e = col_ptr[k + 1];
      for (long long q = b; q < e; ++q) acc = __dsub_rn(acc, __dmul_rn(vals[q], __ldcg(zb + rows[q])));
      zb[k] = acc;
    }
    const unsigned ok = __ballot_sync(kFull, j < le);
    fence_acq_rel();
    __syncwarp();
    if (lane == 0) atomicAdd(&done[L], __popc(ok));
  }
}

// Forward: y[r] = rhs[r] - sum_{k<r} G(r,k) y[k], k ascending, skipping
// y[k] == 0 exactly like the column scatter (solver.cpp:45-52; a skipped term
// is replaced by +0.0, which leaves acc bit-identical); then D^+ (:54-58) into
// yd. rhs[r] = rvec[inv[r]] (permutation in, :40-43).
__global__ void __launch_bounds__(kSweepThreads) sweep_forward_kernel(
    int n, int depth, const int* order, const int* level, const long long* lvl_off, const long long* gt_ptr,
    const int* gt_col, const double* gt_val, const double* diag, const int* inv,
    const double* rvec, double* yf, double* yd, int* done, int* frontier, int* counter,
    unsigned long long* trace) {
  __shared__ double buf[kSweepThreads / 32][kRowBlock];
  const int lane = lane_id();
  double* wbuf = buf[threadIdx.x >> 5];
  // Static round-robin of each level's rows over the persistent warps, levels
  // in sweep order: no claim atomics (a single claim counter capped the wide
  // early levels at the L2 same-address atomic rate).
  const int W = (gridDim.x * blockDim.x) >> 5;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  (void)counter;
  (void)level;
  for (int L = 1; L <= depth; ++L) {
   if (lane_mode(lvl_off, L, W)) {
     lane_level_forward(L, depth, w, W, lane, order, lvl_off, gt_ptr, gt_col, gt_val, diag, inv, rvec,
                        yf, yd, done);
     continue;
   }
   for (long long j = first_row(lvl_off[L], w, W); j < lvl_off[L + 1]; j += W) {
    const int r = order[j];
    if (trace && lane == 0) trace[3 * r + 2] = globaltimer_ns();
    if (L > 1 && lane == 0) wait_level(done, lvl_off, L - 1, -1, depth);
    __syncwarp();
    fence_acq_rel();
    if (trace && lane == 0) trace[3 * r] = globaltimer_ns();
    double acc = rvec[inv[r]];
    const long long b = gt_ptr[r], e = gt_ptr[r + 1];
    for (long long base = b; base < e; base += kRowBlock) {
      const int cnt = static_cast<int>(min(static_cast<long long>(kRowBlock), e - base));
      stage_products(gt_col + base, gt_val + base, yf, cnt, lane, true, wbuf);
      __syncwarp();
      if (lane == 0) acc = serial_sub(acc, wbuf, cnt);
      __syncwarp();
    }
    if (lane == 0) {
      yf[r] = acc;
      const double d = diag[r];
      yd[r] = d > 0.0 ? __ddiv_rn(acc, d) : 0.0;
      if (trace) trace[3 * r + 1] = globaltimer_ns();
      finish_row(done, L);
    }
  }
  }
}

// Backward: z[k] = yd[k] - sum_{r in col k, ascending} G(r,k) z[r] (solver.cpp:60-66).
__global__ void __launch_bounds__(kSweepThreads) sweep_backward_kernel(
    int n, int depth, const int* order, const int* level, const long long* lvl_off,
    const long long* col_ptr, const int* rows, const double* vals, const double* yd, double* zb,
    int* done, int* frontier, int* counter, unsigned long long* trace) {
  __shared__ double buf[kSweepThreads / 32][kRowBlock];
  const int lane = lane_id();
  double* wbuf = buf[threadIdx.x >> 5];
  const int W = (gridDim.x * blockDim.x) >> 5;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  (void)counter;
  (void)level;
  for (int L = depth; L >= 1; --L) {
   if (lane_mode(lvl_off, L, W)) {
     lane_level_backward(L, depth, w, W, lane, order, lvl_off, col_ptr, rows, vals, yd, zb, done);
     continue;
   }
   for (long long j = first_row(lvl_off[L], w, W); j < lvl_off[L + 1]; j += W) {
    const int k = order[j];
    if (trace && lane == 0) trace[3 * k + 2] = globaltimer_ns();
    if (L < depth && lane == 0) wait_level(done, lvl_off, L + 1, +1, depth);
    __syncwarp();
    fence_acq_rel();
    if (trace && lane == 0) trace[3 * k] = globaltimer_ns();
    double acc = yd[k];
    const long long b = col_ptr[k], e = col_ptr[k + 1];
    for (long long base = b; base < e; base += kRowBlock) {
      const int cnt = static_cast<int>(min(static_cast<long long>(kRowBlock), e - base));
      stage_products(rows + base, vals + base, zb, cnt, lane, false, wbuf);
      __syncwarp();
      if (lane == 0) acc = serial_sub(acc, wbuf, cnt);
      __syncwarp();
    }
    if (lane == 0) {
      zb[k] = acc;
      if (trace) trace[3 * k + 1] = globaltimer_ns();
      finish_row(done, L);
    }
  }
  }
}

// ------------------------------------------------------------ K6 (fast mode)
// PCG does not need the reference's summation order (only its iteration count
// and residual, BASELINE north_star), so the default preconditioner for the
// solve sums each row with a fixed per-lane split + warp tree (deterministic,
// run-to-run identical) and -- the point -- consumes a row's entries sorted by
// the level of the value they read: every block of 32 waits only for its own
// latest dependency level, so all but the last block of a row are summed while
// earlier levels are still finishing. After the last dependency lands, a row
// costs one load round trip plus a 5-step tree.
//
// Invariant (both directions): done[X] == size(X) implies every level before X
// in sweep order is complete -- each row of level X reads a value of the
// previous level (ASAP levels), so it cannot finish before that level did.

// Segmented sort of (idx, val) within each segment by key = level-derived u64.
// Warp per segment; <= 32 in registers, longer segments by ranking in place
// through a scratch copy (rare: long rows of the last few hundred levels).
__global__ void level_sort_kernel(int nseg, const long long* seg, const int* idx_in, const double* val_in,
                                  const int* level, int desc, int maxlevel, int* idx_out, double* val_out,
                                  int* lvl_out) {
  const int lane = lane_id();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int sgi = gw; sgi < nseg; sgi += nw) {
    const long long b = seg[sgi];
    const int len = static_cast<int>(seg[sgi + 1] - b);
    auto key_of = [&](int j) -> unsigned long long {
      const int id = idx_in[b + j];
      const int lv = level[id];
      const unsigned hi = desc ? static_cast<unsigned>(maxlevel - lv) : static_cast<unsigned>(lv);
      return (static_cast<unsigned long long>(hi) << 32) | static_cast<unsigned>(id);
    };
    for (int base = 0; base < len; base += 32) {
      const int t = base + lane;
      const unsigned long long mk = t < len ? key_of(t) : ~0ull;
      int rank = 0;
      for (int j = 0; j < len; ++j) rank += key_of(j) < mk;
      if (t < len) {
        idx_out[b + rank] = idx_in[b + t];
        val_out[b + rank] = val_in[b + t];
        lvl_out[b + rank] = level[idx_in[b + t]];
      }
    }
  }
}

// One batch of up to 32*Q entries of a fast-mode row: index/coefficient loads
// first (independent of the wait), then -- once the batch's latest dependency
// level is complete -- all value loads in flight together, then the lane's
// partial sum in fixed order (deterministic).
template <int Q>
__device__ __forceinline__ double fast_batch(const int* idx, const double* g, const double* x, int cnt,
                                             int lane, double part) {
  int ci[Q];
  double gv[Q], xv[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const bool ok = q * 32 + lane < cnt;
    ci[q] = ok ? idx[q * 32 + lane] : 0;
    gv[q] = ok ? g[q * 32 + lane] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) xv[q] = q * 32 + lane < cnt ? __ldcg(x + ci[q]) : 0.0;
#pragma unroll
  for (int q = 0; q < Q; ++q) part += gv[q] * xv[q];
  return part;
}

// Forward, fast: y[r] = rhs[r] - sum G(r,k) y[k]; entries sorted by level[k] ascending.
__global__ void __launch_bounds__(kSweepThreads, 6) sweep_forward_fast_kernel(
    int n, int depth, const int* order, const int* level, const long long* lvl_off, const long long* gt_ptr,
    const int* fcol, const double* fval, const int* flvl, const int* gt_col, const double* gt_val,
    const double* diag, const int* inv, const double* rvec, double* yf, double* yd, int* done, int* counter,
    unsigned long long* trace) {
  const int lane = lane_id();
  // Static round-robin of each level's rows over the persistent warps, levels
  // in sweep order: no claim atomics (a single claim counter capped the wide
  // early levels at the L2 same-address atomic rate).
  const int W = (gridDim.x * blockDim.x) >> 5;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  (void)counter;
  (void)level;
  for (int L = 1; L <= depth; ++L) {
   if (lane_mode(lvl_off, L, W)) {
     lane_level_forward(L, depth, w, W, lane, order, lvl_off, gt_ptr, gt_col, gt_val, diag, inv, rvec,
                        yf, yd, done);
     continue;
   }
   for (long long j = first_row(lvl_off[L], w, W); j < lvl_off[L + 1]; j += W) {
    const int r = order[j];
    if (trace && lane == 0) trace[3 * r + 2] = globaltimer_ns();
    const long long b = gt_ptr[r], e = gt_ptr[r + 1];
    double part = 0.0;
    for (long long base = b; base < e; base += kFastBlock) {
      const int cnt = static_cast<int>(min(static_cast<long long>(kFastBlock), e - base));
      const int need = flvl[base + cnt - 1];  // latest dependency level in the batch
      if (lane == 0) wait_level(done, lvl_off, need, -1, depth);
      __syncwarp();
      fence_acq_rel();
      part = fast_batch<kFastBlock / 32>(fcol + base, fval + base, yf, cnt, lane, part);
    }
    if (trace && lane == 0) trace[3 * r] = globaltimer_ns();
    const double sum = warp_sum(part);
    if (lane == 0) {
      if (trace) trace[3 * r + 1] = globaltimer_ns();
      const double acc = rvec[inv[r]] - sum;
      yf[r] = acc;
      const double d = diag[r];
      yd[r] = d > 0.0 ? acc / d : 0.0;
      finish_row(done, L);
    }
  }
  }
}

// Backward, fast: z[k] = yd[k] - sum G(r,k) z[r]; entries sorted by level[r] descending.
__global__ void __launch_bounds__(kSweepThreads, 6) sweep_backward_fast_kernel(
    int n, int depth, const int* order, const int* level, const long long* lvl_off, const long long* col_ptr,
    const int* brow, const double* bval, const int* blvl, const int* rows, const double* vals,
    const double* yd, double* zb, int* done, int* counter, unsigned long long* trace) {
  const int lane = lane_id();
  const int W = (gridDim.x * blockDim.x) >> 5;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  (void)counter;
  (void)level;
  for (int L = depth; L >= 1; --L) {
   if (lane_mode(lvl_off, L, W)) {
     lane_level_backward(L, depth, w, W, lane, order, lvl_off, col_ptr, rows, vals, yd, zb, done);
     continue;
   }
   for (long long j = first_row(lvl_off[L], w, W); j < lvl_off[L + 1]; j += W) {
    const int k = order[j];
    if (trace && lane == 0) trace[3 * k + 2] = globaltimer_ns();
    const long long b = col_ptr[k], e = col_ptr[k + 1];
    double part = 0.0;
    for (long long base = b; base < e; base += kFastBlock) {
      const int cnt = static_cast<int>(min(static_cast<long long>(kFastBlock), e - base));
      const int need = blvl[base + cnt - 1];
      if (lane == 0) wait_level(done, lvl_off, need, +1, depth);
      __syncwarp();
      fence_acq_rel();
      part = fast_batch<kFastBlock / 32>(brow + base, bval + base, zb, cnt, lane, part);
    }
    if (trace && lane == 0) trace[3 * k] = globaltimer_ns();
    const double sum = warp_sum(part);
    if (lane == 0) {
      if (trace) trace[3 * k + 1] = globaltimer_ns();
      zb[k] = yd[k] - sum;
      finish_row(done, L);
    }
  }
  }
}

// Persistent sweep grids: exactly the co-resident capacity of each kernel.
// The static row assignment needs every CTA resident (a non-resident CTA's
// rows would never run while resident ones wait on their level), so each
// kernel is sized from its own occupancy (register/smem use differ).
template <typename K>
int occupancy_grid(K kernel, int device) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kSweepThreads, 0);
  return std::max(1, per_sm) * sm_count(device);
}

struct SweepGrids {
  int fwd, bwd, fwd_fast, bwd_fast, level;
};

SweepGrids sweep_grids(int device) {
  static SweepGrids cached[64] = {};
  if (device >= 0 && device < 64 && cached[device].fwd) return cached[device];
  SweepGrids g{occupancy_grid(sweep_forward_kernel, device), occupancy_grid(sweep_backward_kernel, device),
               occupancy_grid(sweep_forward_fast_kernel, device),
               occupancy_grid(sweep_backward_fast_kernel, device), occupancy_grid(level_kernel, device)};
  if (device >= 0 && device < 64) cached[device] = g;
  return g;
}

int sweep_grid(int device) { return sweep_grids(device).level; }

// ---------------------------------------------------------------- host side
void ensure_vectors(SolveState& s, int n) {
  if (s.cap_n >= static_cast<std::size_t>(n) && s.x) return;
  const std::size_t c = static_cast<std::size_t>(std::max(n, 1));
  dalloc(s.x, c); dalloc(s.r, c); dalloc(s.p, c); dalloc(s.lp, c); dalloc(s.z, c);
  dalloc(s.best, c); dalloc(s.yf, c); dalloc(s.yd, c); dalloc(s.zb, c); dalloc(s.rhs, c);
  dalloc(s.wdeg, c); dalloc(s.inv, c); dalloc(s.level, c); dalloc(s.order, c);
  dalloc(s.flags, c); dalloc(s.tmp_int, c + 2); dalloc(s.done, 2 * c + 8);
  if (std::getenv("PARAC_SWEEP_TRACE")) dalloc(s.trace, 6 * c);  // diagnostics only
  dalloc(s.partials, static_cast<std::size_t>(kRedBlocks) * kSlots);
  dalloc(s.scalars, kScalars);
  dalloc(s.counters, 16);
  dalloc(s.gt_ptr, c + 1);
  dalloc(s.lvl_off, c + 2);
  dalloc(s.tiles, static_cast<std::size_t>(scan_tiles(n) + 2));
  s.cap_n = c;
  s.graph_ready = false;
  s.factor_ready = false;
  s.epoch = 0;
  check(cudaMemset(s.flags, 0, c * sizeof(int)), "memset");
}

void prepare_graph(const SolveInputs& in) {
  SolveState& s = *in.state;
  ensure_vectors(s, in.n);
  if (s.graph_ready && s.n == in.n) return;
  const int n = in.n;
  const int blocks = (n + 255) / 256;
  cudaStream_t st = in.stream;
  wdeg_kernel<<<blocks, 256, 0, st>>>(n, in.ptr, in.w, s.wdeg);
  note_launches(1);
  s.n = n;
  s.graph_ready = true;
  check(cudaGetLastError(), "wdeg");
}

int component_count(const SolveInputs& in) {
  SolveState& s = *in.state;
  const int n = in.n;
  if (n == 0) return 0;
  const int blocks = (n + 255) / 256;
  cudaStream_t st = in.stream;
  int* parent = s.tmp_int;
  int* count = s.counters + 8;
  check(cudaMemsetAsync(count, 0, sizeof(int), st), "memset");
  cc_init<<<blocks, 256, 0, st>>>(n, parent);
  cc_hook<<<blocks, 256, 0, st>>>(n, in.ptr, in.adj, parent);
  cc_count_roots<<<blocks, 256, 0, st>>>(n, parent, count);
  note_launches(3);
  int h = 0;
  check(cudaMemcpyAsync(&h, count, sizeof(int), cudaMemcpyDeviceToHost, st), "cc");
  check(cudaStreamSynchronize(st), "cc sync");
  return h;
}

void prepare_factor(const SolveInputs& in) {
  SolveState& s = *in.state;
  if (s.factor_ready) return;
  const int n = in.f_n;
  const long long Z = in.f_nnz;
  cudaStream_t st = in.stream;
  const int blocks = (n + 255) / 256;
  const int sms = sm_count(in.device);
  if (s.cap_z < static_cast<std::size_t>(std::max<long long>(Z, 1))) {
    const std::size_t cz = static_cast<std::size_t>(std::max<long long>(Z, 1));
    dalloc(s.gt_col, cz);
    dalloc(s.gt_val, cz);
    dalloc(s.ff_col, cz);
    dalloc(s.ff_val, cz);
    dalloc(s.ff_lvl, cz);
    dalloc(s.fb_row, cz);
    dalloc(s.fb_val, cz);
    dalloc(s.fb_lvl, cz);
    s.cap_z = static_cast<std::size_t>(std::max<long long>(Z, 1));
  }
  inverse_perm_kernel<<<blocks, 256, 0, st>>>(n, in.perm, s.inv);
  int* cnt = s.tmp_int;
  check(cudaMemsetAsync(cnt, 0, sizeof(int) * (n + 1), st), "memset");
  gt_count_kernel<<<sms * 4, 256, 0, st>>>(Z, in.rows, cnt);
  note_launches(2);
  check(launch_scan(cnt, n, s.gt_ptr, s.tiles, st), "scan");
  check(cudaMemsetAsync(cnt, 0, sizeof(int) * (n + 1), st), "memset");
  gt_fill_kernel<<<sms * 8, 256, 0, st>>>(n, in.col_ptr, in.rows, in.vals, s.gt_ptr, cnt, s.gt_col, s.gt_val);
  gt_sort_kernel<<<sms * 8, 256, 0, st>>>(n, s.gt_ptr, s.gt_col, s.gt_val);
  note_launches(2);
  // levels: recorded by the elimination kernel for factors computed here,
  // recomputed (sync-free pass over G's rows) for uploaded ones
  check(cudaMemsetAsync(s.counters, 0, sizeof(int) * 4, st), "memset");
  if (in.level) {
    check(cudaMemcpyAsync(s.level, in.level, sizeof(int) * n, cudaMemcpyDeviceToDevice, st), "d2d");
  } else {
    const int stamp = ++s.epoch;
    level_kernel<<<sweep_grid(in.device), kSweepThreads, 0, st>>>(n, s.gt_ptr, s.gt_col, s.level,
                                                                  s.flags, stamp, s.counters);
    note_launches(1);
  }
  // counting sort of positions by level
  int* hist = s.tmp_int;  // levels are 1..n
  check(cudaMemsetAsync(hist, 0, sizeof(int) * (n + 2), st), "memset");
  level_hist_kernel<<<blocks, 256, 0, st>>>(n, s.level, hist, s.counters + 1);
  note_launches(2);
  check(launch_scan(hist, n + 1, s.lvl_off, s.tiles, st), "scan");
  check(cudaMemsetAsync(hist, 0, sizeof(int) * (n + 2), st), "memset");  // reuse as cursor
  level_scatter_kernel<<<blocks, 256, 0, st>>>(n, s.level, s.lvl_off, hist, s.order);
  note_launches(1);
  int depth = 0;
  check(cudaMemcpyAsync(&depth, s.counters + 1, sizeof(int), cudaMemcpyDeviceToHost, st), "d2h");
  check(cudaStreamSynchronize(st), "prepare_factor");
  s.depth = depth;
  // fast-mode copies: G rows sorted by level[k] ascending, G columns by level[r] descending
  level_sort_kernel<<<sms * 8, 256, 0, st>>>(n, s.gt_ptr, s.gt_col, s.gt_val, s.level, 0, depth + 1,
                                             s.ff_col, s.ff_val, s.ff_lvl);
  level_sort_kernel<<<sms * 8, 256, 0, st>>>(n, in.col_ptr, in.rows, in.vals, s.level, 1, depth + 1,
                                             s.fb_row, s.fb_val, s.fb_lvl);
  note_launches(2);
  check(cudaGetLastError(), "level sort");
  s.factor_ready = true;
}

double host_sum(const std::vector<double>& v) {
  double s = 0.0;
  for (double x : v) s += x;  // same order as sum_partials on the device
  return s;
}

struct Solver {
  const SolveInputs& in;
  SolveState& s;
  cudaStream_t st;
  int n;
  SweepGrids grids;
  std::vector<double> hp = std::vector<double>(kRedBlocks);

  explicit Solver(const SolveInputs& i)
      : in(i), s(*i.state), st(i.stream), n(i.n), grids(sweep_grids(i.device)) {}

  double* part(int slot) const { return s.partials + slot * kRedBlocks; }

  double read_partials(int slot) {
    check(cudaMemcpyAsync(hp.data(), part(slot), sizeof(double) * kRedBlocks,
                          cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaStreamSynchronize(st), "sync");
    return host_sum(hp);
  }

  // z (label space) = M^-1 r (label space); partial r.z into slot.
  void precond(const double* r, double* z, int slot, bool exact = true) {
    const int D = s.depth;
    int* done_f = s.done;
    int* done_b = s.done + (D + 2);
    check(cudaMemsetAsync(s.done, 0, sizeof(int) * 2 * (D + 2), st), "memset");
    check(cudaMemsetAsync(s.counters + 2, 0, sizeof(int) * 4, st), "memset");
    if (!exact) {
      sweep_forward_fast_kernel<<<grids.fwd_fast, kSweepThreads, 0, st>>>(
          in.f_n, D, s.order, s.level, s.lvl_off, s.gt_ptr, s.ff_col, s.ff_val, s.ff_lvl, s.gt_col,
          s.gt_val, in.diag, s.inv, r, s.yf, s.yd, done_f, s.counters + 2, s.trace);
      sweep_backward_fast_kernel<<<grids.bwd_fast, kSweepThreads, 0, st>>>(
          in.f_n, D, s.order, s.level, s.lvl_off, in.col_ptr, s.fb_row, s.fb_val, s.fb_lvl, in.rows,
          in.vals, s.yd, s.zb, done_b, s.counters + 3, s.trace ? s.trace + 3 * in.f_n : nullptr);
      gather_z_dot_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(in.f_n, in.perm, s.zb, r, z, part(slot));
      note_launches(3);
      return;
    }
    sweep_forward_kernel<<<grids.fwd, kSweepThreads, 0, st>>>(
        in.f_n, D, s.order, s.level, s.lvl_off, s.gt_ptr, s.gt_col, s.gt_val, in.diag, s.inv, r,
        s.yf, s.yd, done_f, s.counters + 4, s.counters + 2, s.trace);
    sweep_backward_kernel<<<grids.bwd, kSweepThreads, 0, st>>>(
        in.f_n, D, s.order, s.level, s.lvl_off, in.col_ptr, in.rows, in.vals, s.yd, s.zb, done_b,
        s.counters + 5, s.counters + 3, s.trace ? s.trace + 3 * in.f_n : nullptr);
    gather_z_dot_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(in.f_n, in.perm, s.zb, r, z, part(slot));
    note_launches(3);
  }

  // The sweeps' abort words (done[0] of each direction, see wait_level).
  void check_abort() {
    int flags[2] = {0, 0};
    check(cudaMemcpyAsync(&flags[0], s.done, sizeof(int), cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaMemcpyAsync(&flags[1], s.done + (s.depth + 2), sizeof(int), cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaStreamSynchronize(st), "sync");
    if (flags[0] || flags[1])
      throw Failure{queue_stall, "triangular sweep made no progress for 20 s (watchdog)"};
  }

  void spmv(const double* x, double* y, int slot) {
    spmv_dot_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, in.ptr, in.adj, in.w, s.wdeg, x, y, part(slot));
    note_launches(1);
  }

  // subtract_mean in place; returns ||a||^2 partial slot B filled
  void center(const double* a, double* out, double* r, double* x) {
    sum_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, a, part(kSlotA));
    center_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, a, part(kSlotA), out, r, x, part(kSlotB));
    note_launches(2);
  }
};

void upload(double* dst, const double* src, int n, cudaStream_t st) {
  check(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyHostToDevice, st), "h2d");
}
void download(double* dst, const double* src, int n, cudaStream_t st) {
  check(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "d2h");
  check(cudaStreamSynchronize(st), "d2h sync");
}

// Diagnostics (PARAC_SWEEP_TRACE=<file>): per-position start/end of the last
// forward and backward sweeps, levels and level order, as raw little-endian arrays.
void dump_sweep_trace(const SolveInputs& in, const char* path) {
  const int n = in.f_n;
  std::vector<unsigned long long> tr(6 * static_cast<std::size_t>(n));
  std::vector<int> lv(n);
  check(cudaMemcpy(tr.data(), in.state->trace, tr.size() * 8, cudaMemcpyDeviceToHost), "d2h");
  check(cudaMemcpy(lv.data(), in.state->level, lv.size() * 4, cudaMemcpyDeviceToHost), "d2h");
  FILE* f = std::fopen(path, "wb");
  if (!f) return;
  std::fwrite(&n, 4, 1, f);
  std::fwrite(tr.data(), 8, tr.size(), f);
  std::fwrite(lv.data(), 4, lv.size(), f);
  std::fclose(f);
}

void need_graph(const SolveInputs& in) {
  if (in.n < 0) throw Failure{dimension_mismatch, "no graph staged (call parac_gpu_upload)"};
}
void need_factor(const SolveInputs& in) {
  if (in.f_n < 0) throw Failure{dimension_mismatch, "no resident factor"};
}

}  // namespace

void solve_release(SolveState& s) {
  dfree(s.wdeg); dfree(s.inv); dfree(s.gt_ptr); dfree(s.gt_col); dfree(s.gt_val);
  dfree(s.level); dfree(s.order); dfree(s.done); dfree(s.trace);
  dfree(s.ff_col); dfree(s.ff_val); dfree(s.ff_lvl); dfree(s.fb_row); dfree(s.fb_val); dfree(s.fb_lvl); dfree(s.lvl_off); dfree(s.flags); dfree(s.x); dfree(s.r); dfree(s.p);
  dfree(s.lp); dfree(s.z); dfree(s.best); dfree(s.yf); dfree(s.yd); dfree(s.zb); dfree(s.rhs);
  dfree(s.partials); dfree(s.scalars); dfree(s.counters); dfree(s.tiles); dfree(s.tmp_int);
  s = SolveState{};
}
void solve_invalidate(SolveState& s) {
  s.graph_ready = false;
  s.factor_ready = false;
}
void solve_invalidate_factor(SolveState& s) { s.factor_ready = false; }

}  // namespace parac_gpu

// ------------------------------------------------------------------ C ABI
using namespace parac_gpu;

namespace {

struct WallTimer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double ms() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
};

void ensure_for(const SolveInputs& in) {
  const int need = std::max(in.n, in.f_n);
  ensure_vectors(*in.state, need);
}

}  // namespace

extern "C" {

int parac_gpu_laplacian_apply(parac_gpu_ctx* ctx, const double* x, double* y) {
  return guarded([&] {
    ctx_activate(ctx);
    SolveInputs in = solve_inputs(ctx);
    need_graph(in);
    ensure_for(in);
    prepare_graph(in);
    Solver sv(in);
    upload(in.state->p, x, in.n, in.stream);
    sv.spmv(in.state->p, in.state->lp, kSlotA);
    check(cudaGetLastError(), "spmv");
    download(y, in.state->lp, in.n, in.stream);
  });
}

int parac_gpu_apply_preconditioner(parac_gpu_ctx* ctx, const double* r, double* z) {
  return guarded([&] {
    ctx_activate(ctx);
    SolveInputs in = solve_inputs(ctx);
    need_factor(in);
    ensure_for(in);
    prepare_factor(in);
    Solver sv(in);
    upload(in.state->r, r, in.f_n, in.stream);
    sv.precond(in.state->r, in.state->z, kSlotC, in.state->mode != kModeFast);
    check(cudaGetLastError(), "precond");
    download(z, in.state->z, in.f_n, in.stream);
    sv.check_abort();
    if (in.state->trace) dump_sweep_trace(in, std::getenv("PARAC_SWEEP_TRACE"));
  });
}

int parac_gpu_set_preconditioner_mode(parac_gpu_ctx* ctx, int32_t mode) {
  return guarded([&] {
    ctx_activate(ctx);
    if (mode < 0 || mode > 2) throw Failure{internal_error, "mode must be 0 (default), 1 (exact) or 2 (fast)"};
    solve_inputs(ctx).state->mode = mode;
  });
}

int parac_gpu_schedule_levels(parac_gpu_ctx* ctx, int32_t* levels, int32_t* depth) {
  return guarded([&] {
    ctx_activate(ctx);
    SolveInputs in = solve_inputs(ctx);
    need_factor(in);
    ensure_for(in);
    prepare_factor(in);
    if (levels && in.f_n > 0) {
      check(cudaMemcpyAsync(levels, in.state->level, sizeof(int) * in.f_n, cudaMemcpyDeviceToHost,
                            in.stream), "d2h");
      check(cudaStreamSynchronize(in.stream), "sync");
    }
    if (depth) *depth = in.state->depth;
  });
}

// pcg_solve, src/solver.cpp:95-175.
int parac_gpu_pcg(parac_gpu_ctx* ctx, const double* b, double tol, int32_t max_iters, double* x,
                  parac_gpu_solve_report* report) {
  WallTimer wall;
  return guarded([&] {
    ctx_activate(ctx);
    SolveInputs in = solve_inputs(ctx);
    need_graph(in);
    need_factor(in);
    if (in.f_n != in.n) throw Failure{dimension_mismatch, "solver inputs disagree on size"};
    ensure_for(in);
    prepare_graph(in);
    if (component_count(in) > 1) throw Failure{not_connected, "pcg requires a connected graph"};
    prepare_factor(in);
    SolveState& s = *in.state;
    const int n = in.n;
    cudaStream_t st = in.stream;
    Solver sv(in);
    parac_gpu_solve_report rep{};
    cudaEvent_t e0, e1;
    check(cudaEventCreate(&e0), "event");
    check(cudaEventCreate(&e1), "event");
    check(cudaEventRecord(e0, st), "event");

    upload(s.lp, b, n, st);
    sv.center(s.lp, s.rhs, s.r, s.x);  // rhs = b - mean, r = rhs, x = 0
    const double b_norm = std::sqrt(sv.read_partials(kSlotB));
    if (b_norm == 0.0) {
      rep.converged = 1;
    } else {
      sv.precond(s.r, s.z, kSlotC, s.mode == kModeExact);
      update_p_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, sv.part(kSlotC), s.scalars, kRz0, kRz0, 1, s.z, s.p);
      copy_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, s.x, s.best);
      note_launches(2);
      double best_norm = b_norm;  // norm2(r) with r = rhs
      double rn = b_norm;
      int iters = 0, slot = kRz0;
      std::vector<double> flag(1);
      while (iters < max_iters) {
        if (rn <= tol * b_norm) break;
        ++iters;
        sv.spmv(s.p, s.lp, kSlotA);
        update_xr_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, sv.part(kSlotA), s.scalars, slot, s.x, s.r,
                                                             s.p, s.lp, sv.part(kSlotB), s.scalars + kPlpOk);
        note_launches(1);
        check(cudaMemcpyAsync(flag.data(), s.scalars + kPlpOk, sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
        const double rr = sv.read_partials(kSlotB);
        if (flag[0] == 0.0) break;  // numerically exhausted search direction
        rn = std::sqrt(rr);
        if (rn < best_norm) {
          best_norm = rn;
          copy_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, s.x, s.best);
          note_launches(1);
        }
        sv.precond(s.r, s.z, kSlotC, s.mode == kModeExact);
        const int next = slot == kRz0 ? kRz1 : kRz0;
        update_p_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, sv.part(kSlotC), s.scalars, slot, next, 0, s.z, s.p);
        note_launches(1);
        slot = next;
      }
      double rec = rn;
      if (rec > best_norm) {
        copy_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, s.best, s.x);
        note_launches(1);
        rec = best_norm;
      }
      rep.recurrence_residual = rec / b_norm;
      sv.center(s.x, s.x, nullptr, nullptr);  // subtract_mean(x)
      sv.spmv(s.x, s.lp, kSlotA);
      diff_norm_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, s.rhs, s.lp, sv.part(kSlotB));
      note_launches(1);
      rep.iterations = iters;
      rep.relative_residual = std::sqrt(sv.read_partials(kSlotB)) / b_norm;
      rep.converged = rep.relative_residual <= tol;
    }
    check(cudaEventRecord(e1, st), "event");
    check(cudaGetLastError(), "pcg");
    if (b_norm != 0.0) sv.check_abort();
    download(x, s.x, n, st);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    rep.solve_ms = ms;
    rep.wall_ms = wall.ms();
    if (report) *report = rep;
  });
}

}  // extern "C"
