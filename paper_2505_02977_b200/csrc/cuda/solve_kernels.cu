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
// Forward: y[r] = rhs[r] - sum_{k<r} G(r,k) y[k], k ascending, skipping y[k]==0
// exactly like the column scatter (solver.cpp:45-52); then the D^+ step
// (:54-58) writes yd[r]. rhs[r] = rvec[inv[r]] (permutation in, :40-43).
__global__ void __launch_bounds__(kSweepThreads) sweep_forward_kernel(
    int n, const int* order, const long long* gt_ptr, const int* gt_col, const double* gt_val,
    const double* diag, const int* inv, const double* rvec, double* yf, double* yd, int* flags,
    int stamp, int* counter) {
  const int lane = lane_id();
  while (true) {
    int i = 0;
    if (lane == 0) i = atomicAdd(counter, 1);
    i = __shfl_sync(kFull, i, 0);
    if (i >= n) return;
    const int r = order[i];
    double acc = rvec[inv[r]];
    const long long b = gt_ptr[r], e = gt_ptr[r + 1];
    for (long long base = b; base < e; base += 32) {
      const long long t = base + lane;
      double prod = 0.0;
      bool use = false;
      int k = 0;
      if (t < e) {
        k = gt_col[t];
        wait_stamp(&flags[k], stamp);
      }
      fence_acq_rel();
      if (t < e) {
        const double yk = __ldcg(yf + k);
        use = yk != 0.0;
        prod = __dmul_rn(gt_val[t], yk);
      }
      const int cnt = static_cast<int>(min(32ll, e - base));
      for (int j = 0; j < cnt; ++j) {
        const double pj = __shfl_sync(kFull, prod, j);
        const bool uj = __shfl_sync(kFull, use, j);
        if (uj) acc = __dsub_rn(acc, pj);
      }
    }
    if (lane == 0) {
      yf[r] = acc;
      const double d = diag[r];
      yd[r] = d > 0.0 ? __ddiv_rn(acc, d) : 0.0;
      st_release(&flags[r], stamp);
    }
  }
}

// Backward: z[k] = yd[k] - sum_{r in col k, ascending} G(r,k) z[r] (solver.cpp:60-66).
__global__ void __launch_bounds__(kSweepThreads) sweep_backward_kernel(
    int n, const int* order, const long long* col_ptr, const int* rows, const double* vals,
    const double* yd, double* zb, int* flags, int stamp, int* counter) {
  const int lane = lane_id();
  while (true) {
    int i = 0;
    if (lane == 0) i = atomicAdd(counter, 1);
    i = __shfl_sync(kFull, i, 0);
    if (i >= n) return;
    const int k = order[n - 1 - i];
    double acc = yd[k];
    const long long b = col_ptr[k], e = col_ptr[k + 1];
    for (long long base = b; base < e; base += 32) {
      const long long t = base + lane;
      double prod = 0.0;
      int r = 0;
      if (t < e) {
        r = rows[t];
        wait_stamp(&flags[r], stamp);
      }
      fence_acq_rel();
      if (t < e) prod = __dmul_rn(vals[t], __ldcg(zb + r));
      const int cnt = static_cast<int>(min(32ll, e - base));
      for (int j = 0; j < cnt; ++j) acc = __dsub_rn(acc, __shfl_sync(kFull, prod, j));
    }
    if (lane == 0) {
      zb[k] = acc;
      st_release(&flags[k], stamp);
    }
  }
}

int sweep_grid(int device) {
  static int cached[64] = {0};
  if (device >= 0 && device < 64 && cached[device]) return cached[device];
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_forward_kernel, kSweepThreads, 0);
  int per_sm_b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_b, sweep_backward_kernel, kSweepThreads, 0);
  per_sm = std::max(1, std::min(per_sm, per_sm_b));
  const int g = per_sm * sm_count(device);
  if (device >= 0 && device < 64) cached[device] = g;
  return g;
}

// ---------------------------------------------------------------- host side
void ensure_vectors(SolveState& s, int n) {
  if (s.cap_n >= static_cast<std::size_t>(n) && s.x) return;
  const std::size_t c = static_cast<std::size_t>(std::max(n, 1));
  dalloc(s.x, c); dalloc(s.r, c); dalloc(s.p, c); dalloc(s.lp, c); dalloc(s.z, c);
  dalloc(s.best, c); dalloc(s.yf, c); dalloc(s.yd, c); dalloc(s.zb, c); dalloc(s.rhs, c);
  dalloc(s.wdeg, c); dalloc(s.inv, c); dalloc(s.level, c); dalloc(s.order, c);
  dalloc(s.flags, c); dalloc(s.tmp_int, c + 2);
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
    dalloc(s.gt_col, static_cast<std::size_t>(std::max<long long>(Z, 1)));
    dalloc(s.gt_val, static_cast<std::size_t>(std::max<long long>(Z, 1)));
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
  // levels
  const int stamp = ++s.epoch;
  check(cudaMemsetAsync(s.counters, 0, sizeof(int) * 4, st), "memset");
  level_kernel<<<sweep_grid(in.device), kSweepThreads, 0, st>>>(n, s.gt_ptr, s.gt_col, s.level,
                                                                s.flags, stamp, s.counters);
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
  int sweep_blocks;
  std::vector<double> hp = std::vector<double>(kRedBlocks);

  explicit Solver(const SolveInputs& i)
      : in(i), s(*i.state), st(i.stream), n(i.n), sweep_blocks(sweep_grid(i.device)) {}

  double* part(int slot) const { return s.partials + slot * kRedBlocks; }

  double read_partials(int slot) {
    check(cudaMemcpyAsync(hp.data(), part(slot), sizeof(double) * kRedBlocks,
                          cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaStreamSynchronize(st), "sync");
    return host_sum(hp);
  }

  // z (label space) = M^-1 r (label space); partial r.z into slot.
  void precond(const double* r, double* z, int slot) {
    const int f_stamp = ++s.epoch;
    const int b_stamp = ++s.epoch;
    check(cudaMemsetAsync(s.counters + 2, 0, sizeof(int) * 2, st), "memset");
    sweep_forward_kernel<<<sweep_blocks, kSweepThreads, 0, st>>>(
        in.f_n, s.order, s.gt_ptr, s.gt_col, s.gt_val, in.diag, s.inv, r, s.yf, s.yd, s.flags,
        f_stamp, s.counters + 2);
    sweep_backward_kernel<<<sweep_blocks, kSweepThreads, 0, st>>>(
        in.f_n, s.order, in.col_ptr, in.rows, in.vals, s.yd, s.zb, s.flags, b_stamp,
        s.counters + 3);
    gather_z_dot_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(in.f_n, in.perm, s.zb, r, z, part(slot));
    note_launches(3);
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

void need_graph(const SolveInputs& in) {
  if (in.n < 0) throw Failure{dimension_mismatch, "no graph staged (call parac_gpu_upload)"};
}
void need_factor(const SolveInputs& in) {
  if (in.f_n < 0) throw Failure{dimension_mismatch, "no resident factor"};
}

}  // namespace

void solve_release(SolveState& s) {
  dfree(s.wdeg); dfree(s.inv); dfree(s.gt_ptr); dfree(s.gt_col); dfree(s.gt_val);
  dfree(s.level); dfree(s.order); dfree(s.lvl_off); dfree(s.flags); dfree(s.x); dfree(s.r); dfree(s.p);
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
    sv.precond(in.state->r, in.state->z, kSlotC);
    check(cudaGetLastError(), "precond");
    download(z, in.state->z, in.f_n, in.stream);
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
      sv.precond(s.r, s.z, kSlotC);
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
        sv.precond(s.r, s.z, kSlotC);
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
