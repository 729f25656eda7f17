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
#include "../host/nvtx.hpp"
#include "common.cuh"
#include "factor_kernels.cuh"
#include "solve_kernels.cuh"
#include "radix_sort.cuh"

namespace parac_gpu {

void note_launches(long long k);

using namespace dev;

namespace {

constexpr int kRedBlocks = 296;  // 2 x 148 SMs: fixed => deterministic reductions
constexpr int kRedThreads = 256;
constexpr int kSweepThreads = 256;

enum Slot { kSlotA = 0, kSlotB = 1, kSlotC = 2, kSlots = 3 };
enum Scalar { kRz0 = 0, kRz1 = 1, kPlpOk = 2, kRzPrev = 6, kRn = 7, kBest = 8, kTolB = 9, kScalars = 16 };
// int control words of the fast PCG loop (SolveState::counters + kCtl): iterations, max_iters, copy-best flag
enum Ctl { kCtl = 12, kCtlIters = 0, kCtlMax = 1, kCtlCopy = 2 };

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
    } else if (len <= 256) {
      // up to 8 keys per lane, ranked against every key of the row (keys are
      // unique columns) through register broadcasts; then scattered in place
      int k[8];
      double v[8];
      int rank[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = i * 32 + lane;
        k[i] = e < len ? gt_col[b + e] : 0x7fffffff;
        v[i] = e < len ? gt_val[b + e] : 0.0;
        rank[i] = 0;
      }
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        if (jj * 32 >= len) break;
        for (int src = 0; src < 32; ++src) {
          const int kj = __shfl_sync(kFull, k[jj], src);
#pragma unroll
          for (int i = 0; i < 8; ++i) rank[i] += kj < k[i];
        }
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i * 32 + lane < len) {
          gt_col[b + rank[i]] = k[i];
          gt_val[b + rank[i]] = v[i];
        }
    }  // longer rows: gt_long_* + a CUB segmented sort (prepare_factor)
  }
}

// Rows of G^T longer than 256 entries (hub columns of the factor) are sorted
// out of line: flagged and counted, copied into a compact buffer, sorted there
// by CUB's segmented sort (any length), and copied back.
constexpr int kGtShortRow = 256;
__global__ void gt_long_flags_kernel(int n, const long long* gt_ptr, int* flag, int* len) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const long long l = gt_ptr[r + 1] - gt_ptr[r];
  flag[r] = l > kGtShortRow ? 1 : 0;
  len[r] = l > kGtShortRow ? static_cast<int>(l) : 0;
}
__global__ void gt_long_gather_kernel(int n, const long long* gt_ptr, const int* flag, const long long* rpos,
                                      const long long* loff, const int* gt_col, const double* gt_val, int* beg,
                                      int* end, int* rows, int* ck, double* cv) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = gw; r < n; r += nw) {
    if (!flag[r]) continue;
    const long long b = gt_ptr[r], l = gt_ptr[r + 1] - b, o = loff[r];
    if (lane == 0) {
      const long long i = rpos[r];
      beg[i] = static_cast<int>(o);
      end[i] = static_cast<int>(o + l);
      rows[i] = r;
    }
    for (long long q = lane; q < l; q += 32) {
      ck[o + q] = gt_col[b + q];
      cv[o + q] = gt_val[b + q];
    }
  }
}
// Long rows sorted by one radix sort over all of them: key (row slot << cb) |
// column, value = entry index; the slots are contiguous in [beg, end) order,
// so the sorted sequence lands back in each row's own range.
__global__ void gt_long_keys_kernel(int nl, const int* beg, const int* end, const int* ck, int cb,
                                    unsigned long long* key, int* idx) {
  for (int i = blockIdx.x; i < nl; i += gridDim.x)
    for (int t = beg[i] + threadIdx.x; t < end[i]; t += blockDim.x) {
      key[t] = (static_cast<unsigned long long>(i) << cb) | static_cast<unsigned>(ck[t]);
      idx[t] = t;
    }
}

__global__ void gt_long_unkey_kernel(long long T, const unsigned long long* key, const int* idx, unsigned long long cmask,
                                     const double* cv, int* ck2, double* cv2) {
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < T;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    ck2[t] = static_cast<int>(key[t] & cmask);
    cv2[t] = cv[idx[t]];
  }
}

__global__ void gt_long_scatter_kernel(int nl, const long long* gt_ptr, const int* beg, const int* end,
                                       const int* rows, const int* ck, const double* cv, int* gt_col,
                                       double* gt_val) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < nl; i += nw) {
    const long long b = gt_ptr[rows[i]];
    for (int q = beg[i] + lane; q < end[i]; q += 32) {
      gt_col[b + q - beg[i]] = ck[q];
      gt_val[b + q - beg[i]] = cv[q];
    }
  }
}

// Relaxed polling with exponential backoff (no L1 invalidation per poll); the
// caller follows with fence_acq_rel() before reading the producer's data.
// Bounded: after ~`budget_ns` without the stamp (a malformed factor whose
// rows reference a column that is never finished) the wait raises `*abort`
// and returns false; every waiter then bails out instead of hanging the GPU.
__device__ __forceinline__ bool wait_stamp(const int* flag, int stamp, int* abort,
                                           unsigned long long budget_ns = 10000000000ull) {
  if (ld_relaxed(flag) >= stamp) return true;
  unsigned ns = 32;
  const unsigned long long t0 = globaltimer_ns();
  int it = 0;
  do {
    __nanosleep(ns);
    if (ns < 512) ns <<= 1;
    if ((++it & 63) == 0) {
      if (ld_relaxed(abort) != 0) return false;
      if (globaltimer_ns() - t0 > budget_ns) {
        atomicExch(abort, 1);
        return false;
      }
    }
  } while (ld_relaxed(flag) < stamp);
  return true;
}

// ASAP levels of the factor DAG (schedule_levels, src/factor_par.cpp:659-684):
// level[r] = 1 + max level over G's row r. Sync-free, positions claimed in
// ascending order (all dependencies are earlier positions => deadlock-free).
__global__ void level_kernel(int n, const long long* gt_ptr, const int* gt_col, int* level,
                             int* flags, int stamp, int* counter, int* abort) {
  const int lane = lane_id();
  while (true) {
    int r = 0;
    if (lane == 0) r = atomicAdd(counter, 1);
    r = __shfl_sync(kFull, r, 0);
    if (r >= n) return;
    int lv = 0;
    bool ok = true;
    for (long long t = gt_ptr[r] + lane; t < gt_ptr[r + 1]; t += 32) {
      const int k = gt_col[t];
      // uploaded factors are validated (k < r), so this wait is bounded by the
      // DAG; the budget only guards against a corrupted device state
      if (k >= r || !wait_stamp(&flags[k], stamp, abort)) {
        atomicExch(abort, 1);
        ok = false;
        break;
      }
      fence_acq_rel();
      lv = max(lv, ld_relaxed(&level[k]));
    }
    if (!__all_sync(kFull, ok)) return;
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

__global__ void iota_kernel(int n, int* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) out[r] = r;
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

// ---- fast PCG loop, graph form (one iteration = one body of a CUDA-graph
// while node; no host round trip per iteration). The reductions are the same
// fixed-order partial sums as above, read by every block, so every reader
// derives bit-identical scalars.
// Iteration t: rz_{t-1} is partial slot C (r.z of the previous iteration);
// update_xr_g snapshots it into kRzPrev for update_p_g's beta.
__global__ void update_xr_g_kernel(int n, const double* plp_partials, const double* rz_partials, double* scalars,
                                   double* x, double* r, const double* p, const double* lp, double* partials) {
  __shared__ double alpha;
  __shared__ int ok;
  if (threadIdx.x == 0) {
    const double plp = sum_partials(plp_partials);
    const double rz = sum_partials(rz_partials);
    ok = plp > 0.0;  // solver.cpp:134
    alpha = ok ? rz / plp : 0.0;
    if (blockIdx.x == 0) {
      scalars[kPlpOk] = ok ? 1.0 : 0.0;
      scalars[kRzPrev] = rz;
    }
  }
  __syncthreads();
  double s = 0.0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    double rv = r[v];
    if (ok) {
      x[v] = __dadd_rn(x[v], __dmul_rn(alpha, p[v]));  // unfused, as solver.cpp:137-138
      rv = __dsub_rn(rv, __dmul_rn(alpha, lp[v]));
      r[v] = rv;
    }
    s += rv * rv;
  }
  block_partial(s, partials);
}

// The loop test of solver.cpp:129-131 + the best-iterate bookkeeping of
// :141-144, on the device: one thread. Sets the while node's condition.
__global__ void pcg_control_kernel(const double* rr_partials, double* scalars, int* ctl,
                                   cudaGraphConditionalHandle cond, int set_cond) {
  const double rn = sqrt(sum_partials(rr_partials));
  const bool ok = scalars[kPlpOk] != 0.0;
  const int it = ctl[kCtlIters] + 1;  // ++iters precedes the p.Lp test (solver.cpp:132)
  ctl[kCtlIters] = it;
  int copy = 0;
  if (ok) {
    scalars[kRn] = rn;
    if (rn < scalars[kBest]) {
      scalars[kBest] = rn;
      copy = 1;
    }
  }
  ctl[kCtlCopy] = copy;
  const int cont = ok && it < ctl[kCtlMax] && rn > scalars[kTolB];
  if (set_cond) cudaGraphSetConditional(cond, cont ? 1u : 0u);
  ctl[kCtlCopy + 1] = cont;
}

__global__ void copy_if_kernel(int n, const int* flag, const double* a, double* b) {
  if (!*flag) return;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) b[v] = a[v];
}

// beta = rz_t / rz_{t-1}; p = z + beta p (solver.cpp:146-152)
__global__ void update_p_g_kernel(int n, const double* rz_partials, const double* scalars, const double* z,
                                  double* p) {
  __shared__ double beta;
  if (threadIdx.x == 0) beta = sum_partials(rz_partials) / scalars[kRzPrev];
  __syncthreads();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    p[v] = __dadd_rn(z[v], __dmul_rn(beta, p[v]));
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

// ------------------------------------------------ exact PCG (serial chains)
// pcg_solve's reductions are plain left-to-right loops (solver.cpp:15-28):
// dot() is s = fl(s + fl(a_i * b_i)), subtract_mean() sums v_i the same way.
// The exact PCG reproduces them bit for bit: ONE thread runs each chain, the
// other warps of the CTA stream the terms into a double-buffered shared-memory
// stage ahead of it, so the chain runs at the FP64 add latency. Two
// independent chains (e.g. r.r and r.z) interleave in the same thread for the
// price of one. Term kinds:
//   kTermDot:  a_i * b_i        (dot, norm2)
//   kTermSum:  a_i              (subtract_mean)
//   kTermDiff: (a_i - b_i)^2    (norm2 of true_r = rhs - L x, solver.cpp:164-169)
enum : int { kTermDot = 0, kTermSum = 1, kTermDiff = 2 };
struct Chain {
  int kind;
  const double* a;
  const double* b;
};
constexpr int kSerThreads = 256;
constexpr int kSerChunk = 1024;

__device__ __forceinline__ double chain_term(const Chain& c, int i) {
  if (c.kind == kTermSum) return c.a[i];
  if (c.kind == kTermDot) return __dmul_rn(c.a[i], c.b[i]);
  const double t = __dsub_rn(c.a[i], c.b[i]);
  return __dmul_rn(t, t);
}

__global__ void __launch_bounds__(kSerThreads, 1) serial_chain_kernel(int n, Chain c0, Chain c1, int nch,
                                                                      double* out) {
  __shared__ double buf[2][2][kSerChunk];  // [chain][stage][chunk]
  const int tid = threadIdx.x;
  const int nchunks = (n + kSerChunk - 1) / kSerChunk;
  auto fill = [&](int ch, int stage) {
    const int b = ch * kSerChunk, cnt = min(kSerChunk, n - b);
    for (int t = tid - 32; t < cnt; t += kSerThreads - 32) {
      buf[0][stage][t] = chain_term(c0, b + t);
      if (nch > 1) buf[1][stage][t] = chain_term(c1, b + t);
    }
  };
  if (tid >= 32 && nchunks > 0) fill(0, 0);
  double s0 = 0.0, s1 = 0.0;
  for (int ch = 0; ch < nchunks; ++ch) {
    __syncthreads();  // stage ch&1 is full; the other stage is free
    if (tid >= 32) {
      if (ch + 1 < nchunks) fill(ch + 1, (ch + 1) & 1);
    } else if (tid == 0) {
      const double* x0 = buf[0][ch & 1];
      const double* x1 = buf[1][ch & 1];
      const int cnt = min(kSerChunk, n - ch * kSerChunk);
      int t = 0;
      if (nch > 1) {
        for (; t + 8 <= cnt; t += 8) {
          double u[8], v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            u[q] = x0[t + q];
            v[q] = x1[t + q];
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            s0 = __dadd_rn(s0, u[q]);
            s1 = __dadd_rn(s1, v[q]);
          }
        }
        for (; t < cnt; ++t) {
          s0 = __dadd_rn(s0, x0[t]);
          s1 = __dadd_rn(s1, x1[t]);
        }
      } else {
        for (; t + 8 <= cnt; t += 8) {
          double u[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) u[q] = x0[t + q];
#pragma unroll
          for (int q = 0; q < 8; ++q) s0 = __dadd_rn(s0, u[q]);
        }
        for (; t < cnt; ++t) s0 = __dadd_rn(s0, x0[t]);
      }
    }
  }
  if (tid == 0) {
    out[0] = s0;
    if (nch > 1) out[1] = s1;
  }
}

// rhs = b - mean; r = rhs; x = 0 (solver.cpp:107-119, subtract_mean :23-28)
__global__ void center_exact_kernel(int n, const double* a, double mean, double* out, double* r, double* x) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const double o = __dsub_rn(a[v], mean);
    out[v] = o;
    if (r) r[v] = o;
    if (x) x[v] = 0.0;
  }
}

// x += alpha p; r -= alpha lp (solver.cpp:136-139), unfused
__global__ void update_xr_exact_kernel(int n, double alpha, double* x, double* r, const double* p, const double* lp) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    x[v] = __dadd_rn(x[v], __dmul_rn(alpha, p[v]));
    r[v] = __dsub_rn(r[v], __dmul_rn(alpha, lp[v]));
  }
}

// p = z + beta p (solver.cpp:149-152)
__global__ void update_p_exact_kernel(int n, double beta, const double* z, double* p) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    p[v] = __dadd_rn(z[v], __dmul_rn(beta, p[v]));
}

// ------------------------------------------------------------------- K6
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



// Wide levels (>= kLaneRowsPerWarp rows per warp): one row per LANE, summed
// sequentially in the reference's order (so these rows are bit-exact in both
// modes) -- 32 independent rows per warp instead of one keeps the first,
// widest levels (10^5 rows each at 128^3) from being latency-bound per row.






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



// ------------------------------------------------------------ async copy helpers
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Asynchronous L2 prefetch of [p, p + bytes) (16-byte aligned superset), in
// 64 KB bulk requests: the sweeps know every future level's G entries, so
// they pull them from HBM into L2 a few levels ahead of use.
__device__ __forceinline__ void prefetch_l2(const void* p, long long bytes) {
  if (bytes <= 0) return;
  unsigned long long a = reinterpret_cast<unsigned long long>(p) & ~15ull;
  const unsigned long long e = (reinterpret_cast<unsigned long long>(p) + bytes + 15) & ~15ull;
  while (a < e) {
    const unsigned sz = static_cast<unsigned>(min(e - a, 65536ull));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(sz) : "memory");
    a += sz;
  }
}

// ------------------------------------------------------------ K6: cluster sweeps
// One thread-block cluster sweeps levels level-synchronously: every row of
// level L is computed, then ONE hardware cluster barrier (barrier.cluster
// arrive.release / wait.acquire, measured 235 ns on B200 vs ~1.2 us for a
// grid-wide sync) publishes the level. Solution values are written with plain
// stores and read with ld.global.cg (L2), so no stale L1 line can be observed
// after the acquire. Exact mode (cluster_forward/backward_kernel<true>): per-row
// sums in the reference's order (solver.cpp:44-66), lane 0 serial over
// register-staged products -> bit-identical to apply_preconditioner.
constexpr int kCThreads = 1024;
constexpr int kCWarps = kCThreads / 32;
constexpr int kCStage = 128;  // exact mode: products staged per warp before the serial chain

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_nctas() {
  unsigned r;
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}



// Sum of g[q] * x[idx[q]] over [b, e) by one warp.
//   EXACT: acc - p_b - p_{b+1} - ... strictly in order (lane 0), optional
//          zero skip (forward column-scatter semantics: a term with x == 0 is
//          never subtracted, solver.cpp:47-51).
//   FAST:  acc - (fixed-order tree of lane partials).
template <bool EXACT>
__device__ __forceinline__ double warp_row(double acc, const int* idx, const double* g, const double* x,
                                           long long b, long long e, int lane, bool skip_zero,
                                           double* wbuf) {
  if constexpr (!EXACT) {
    double part = 0.0;
    long long q = b + lane;
    for (; q + 96 < e; q += 128) {
      const int c0 = idx[q], c1 = idx[q + 32], c2 = idx[q + 64], c3 = idx[q + 96];
      const double g0 = g[q], g1 = g[q + 32], g2 = g[q + 64], g3 = g[q + 96];
      const double x0 = __ldcg(x + c0), x1 = __ldcg(x + c1), x2 = __ldcg(x + c2), x3 = __ldcg(x + c3);
      part += g0 * x0;
      part += g1 * x1;
      part += g2 * x2;
      part += g3 * x3;
    }
    for (; q < e; q += 32) part += g[q] * __ldcg(x + idx[q]);
    return acc - warp_sum(part);
  } else {
  for (long long base = b; base < e; base += kCStage) {
    const int cnt = static_cast<int>(min(static_cast<long long>(kCStage), e - base));
    constexpr int Q = kCStage / 32;
    int ci[Q];
    double gv[Q], xv[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const bool ok = q * 32 + lane < cnt;
      ci[q] = ok ? idx[base + q * 32 + lane] : 0;
      gv[q] = ok ? g[base + q * 32 + lane] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) xv[q] = q * 32 + lane < cnt ? __ldcg(x + ci[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (q * 32 + lane < cnt) wbuf[q * 32 + lane] = (skip_zero && xv[q] == 0.0) ? 0.0 : __dmul_rn(gv[q], xv[q]);
    __syncwarp();
    if (lane == 0) acc = serial_sub(acc, wbuf, cnt);
    __syncwarp();
  }
  return __shfl_sync(kFull, acc, 0);
  }
}

// One row per lane, serial in the reference's order (exact in both modes).
__device__ __forceinline__ double lane_row(double acc, const int* idx, const double* g, const double* x,
                                           long long b, long long e, bool skip_zero) {
  for (long long q = b; q < e; ++q) {
    const double xv = __ldcg(x + idx[q]);
    if (!(skip_zero && xv == 0.0)) acc = __dsub_rn(acc, __dmul_rn(g[q], xv));
  }
  return acc;
}

// Forward G y = P r over levels 1..H (gather form over G's rows, k ascending),
// then D^+ into yd; afterwards (fast mode with a tail) the G_TH part of every
// tail row: ts_i = rhs_i - sum_{k in H} G(r,k) y_k.
template <bool EXACT>
__global__ void __launch_bounds__(kCThreads, 1) cluster_forward_kernel(
    int H, const long long* lvl_off, const int* order, const long long* gt_ptr, const int* gt_col,
    const double* gt_val, const double* diag, const int* inv, const double* rvec, double* yf, double* yd,
    int nt, int tail_base, const long long* hsplit, const int* ff_col, const double* ff_val, double* ts) {
  __shared__ double stage[EXACT ? kCWarps * kCStage : 1];
  const int lane = lane_id(), wl = threadIdx.x >> 5;
  const int W = static_cast<int>(cluster_nctas()) * kCWarps;
  const int w = static_cast<int>(cluster_rank()) * kCWarps + wl;
  double* wbuf = stage + (EXACT ? wl * kCStage : 0);
  for (int L = 1; L <= H; ++L) {
    const long long lb = lvl_off[L], le = lvl_off[L + 1];
    if (le - lb >= 2LL * W) {
      for (long long j = lb + static_cast<long long>(w) * 32 + lane; j < le; j += 32LL * W) {
        const int r = order[j];
        const double acc = lane_row(rvec[inv[r]], gt_col, gt_val, yf, gt_ptr[r], gt_ptr[r + 1], true);
        yf[r] = acc;
        const double d = diag[r];
        yd[r] = d > 0.0 ? __ddiv_rn(acc, d) : 0.0;
      }
    } else {
      for (long long j = lb + w; j < le; j += W) {
        const int r = order[j];
        const double acc =
            warp_row<EXACT>(rvec[inv[r]], gt_col, gt_val, yf, gt_ptr[r], gt_ptr[r + 1], lane, true, wbuf);
        if (lane == 0) {
          yf[r] = acc;
          const double d = diag[r];
          yd[r] = d > 0.0 ? __ddiv_rn(acc, d) : 0.0;
        }
      }
    }
    cluster_barrier();
  }
  if (!EXACT) {
    for (int i = w; i < nt; i += W) {
      const int r = order[tail_base + i];
      const double acc = warp_row<false>(rvec[inv[r]], ff_col, ff_val, yf, gt_ptr[r], hsplit[i], lane, false, wbuf);
      if (lane == 0) ts[i] = acc;
    }
  }
}

// Backward G^T z = yd over levels H..1 (columns of G, rows ascending); rows of
// higher levels (the tail) are final before launch.
template <bool EXACT>
__global__ void __launch_bounds__(kCThreads, 1) cluster_backward_kernel(
    int H, const long long* lvl_off, const int* order, const long long* col_ptr, const int* rows,
    const double* vals, const double* yd, double* zb) {
  __shared__ double stage[EXACT ? kCWarps * kCStage : 1];
  const int lane = lane_id(), wl = threadIdx.x >> 5;
  const int W = static_cast<int>(cluster_nctas()) * kCWarps;
  const int w = static_cast<int>(cluster_rank()) * kCWarps + wl;
  double* wbuf = stage + (EXACT ? wl * kCStage : 0);
  for (int L = H; L >= 1; --L) {
    const long long lb = lvl_off[L], le = lvl_off[L + 1];
    if (le - lb >= 2LL * W) {
      for (long long j = lb + static_cast<long long>(w) * 32 + lane; j < le; j += 32LL * W) {
        const int k = order[j];
        zb[k] = lane_row(yd[k], rows, vals, zb, col_ptr[k], col_ptr[k + 1], false);
      }
    } else {
      for (long long j = lb + w; j < le; j += W) {
        const int k = order[j];
        const double acc = warp_row<EXACT>(yd[k], rows, vals, zb, col_ptr[k], col_ptr[k + 1], lane, false, wbuf);
        if (lane == 0) zb[k] = acc;
      }
    }
    cluster_barrier();
  }
}

// ---- fast mode, entry-parallel: rows of each level stored contiguously in
// level order (lptr/lidx/lval), each level cut into chunks of whole rows of
// ~equal (entries + rows). A warp takes a chunk, issues ALL of its products'
// loads at once (8 per lane in flight) into a shared-memory product buffer,
// then sums rows from it: lane per row for short rows, warp tree for long
// ones (fixed orders -> run-to-run deterministic). Per level this costs about
// two L2 round trips plus the cluster barrier, instead of (rows per warp) x
// (two dependent round trips).
constexpr int kChunkCap = 768;  // product buffer entries per warp (6 KB; 192 KB per CTA)
constexpr int kShortRow = 16;   // rows up to this length are summed by one lane

template <bool FWD>
__device__ __forceinline__ void finish_row(int j, double s, const int* order, const double* rhs_pos,
                                           const int* inv, const double* rvec, const double* diag, double* x,
                                           double* yd) {
  if constexpr (FWD) {
    const int r = order[j];
    const double acc = rvec[inv[r]] - s;
    x[r] = acc;
    const double d = diag[r];
    yd[r] = d > 0.0 ? acc / d : 0.0;
  } else {
    const int k = order[j];
    x[k] = rhs_pos[k] - s;
  }
}


// ---- v3 head sweep: level-order index space + software pipelining.
// Vectors are indexed by level-order position j (rows of a level are
// contiguous), entry indices are level-order too, and each warp owns exactly
// chunk w of every level (table hrec[L][w] = {jb, je, eb, ee}). While level L
// is computed, the warp already holds level L+1's chunk record and has issued
// the loads of its entries (<= kHeadPF per lane) and row metadata; level
// L+2's record is loaded as well. After the barrier only the gathers of
// solution values (one L2 round trip) remain on the level-to-level chain.
constexpr int kHeadPF = 8;  // entries per lane held in registers (256 per warp)
constexpr int kHThreads = 512;  // 16 warps: 128 registers per thread hold two levels' prefetch
constexpr int kHWarps = kHThreads / 32;
constexpr std::size_t kHeadSmem = static_cast<std::size_t>(kHWarps) * kChunkCap * sizeof(double) + kHWarps * 8 * 16;

struct HeadPre {
  int4 rec;               // jb, je, eb, ee
  int idx[kHeadPF];
  double val[kHeadPF];
  long long rb, re;       // lane's row entry range (absolute; made relative at use, so the
                          // loads issued a level ahead are not waited on here)
  double rhs, dinv;       // lane's row right-hand side and D^+
};

template <bool FWD>
__device__ __forceinline__ void head_load(HeadPre& p, const int4 rec, const long long* lptr, const int* lidx,
                                          const double* lval, const double* rhs_l, const double* dinv_l,
                                          int lane) {
  p.rec = rec;
  const int cnt = rec.w - rec.z;
#pragma unroll
  for (int q = 0; q < kHeadPF; ++q) {
    const int e = q * 32 + lane;
    p.idx[q] = e < cnt ? lidx[rec.z + e] : 0;
    p.val[q] = e < cnt ? lval[rec.z + e] : 0.0;
  }
  const int j = rec.x + lane;
  p.rb = p.re = 0;
  p.rhs = p.dinv = 0.0;
  if (j < rec.y) {
    p.rb = lptr[j];
    p.re = lptr[j + 1];
    p.rhs = rhs_l[j];
    if (FWD) p.dinv = dinv_l[j];
  }
}

// One thread-block cluster sweeps levels Lfirst .. (cluster barrier per level).
// Measured alternatives, removed: a cooperative full-GPU grid for the wide
// levels (grid.sync(); 8-13 us per level, see DESIGN §4 K6); the cluster rows'
// solution in distributed shared memory with the outside operands folded into
// the right-hand side first (no faster: the level time is spread over load
// issue, gathers, row sums and the barrier wait, not the gathers' L2 trip).
template <bool FWD>
__global__ void __launch_bounds__(kHThreads, 1) head_sweep_kernel(
    int Lfirst, int nlev, int W, const int4* hrec, const long long* lptr, const int* lidx, const double* lval,
    const double* rhs_l, const double* dinv_l, double* x, double* yd_l, int nt, int tail_base, double* ts,
    unsigned long long* ltime) {
  extern __shared__ double pbuf_all[];
  const int lane = lane_id(), wl = threadIdx.x >> 5;
  const int w = static_cast<int>(cluster_rank()) * kHWarps + wl;
  double* pbuf = pbuf_all + wl * kChunkCap;
  auto xget = [&](int c) -> double { return __ldcg(x + c); };
  auto xput = [&](int j, double v) { x[j] = v; };
  const double* rhs_rows = rhs_l;
  auto level_barrier = [&]() { cluster_barrier(); };
  auto rec_ptr = [&](int t, int ww) -> const int4* {
    const int L = FWD ? Lfirst + t : Lfirst - t;
    return hrec + static_cast<long long>(L) * W + ww;
  };
  // Chunk records travel through a per-warp shared-memory ring, copied with
  // cp.async kHRing-1 levels ahead (no register waits on them in the loop);
  // the entries of level t+1 are loaded into registers during level t; one
  // thread bulk-prefetches this CTA's slice of level t+4 into L2 (bounds
  // read from the rings of the CTA's first and last warp).
  constexpr int kHRing = 8;
  int4* ring = reinterpret_cast<int4*>(pbuf_all + kHWarps * kChunkCap);  // [kHWarps][kHRing]
  int4* myring = ring + wl * kHRing;
  for (int t = 0; t < kHRing - 1; ++t) {
    if (lane == 0 && t < nlev) cp_async16(&myring[t % kHRing], rec_ptr(t, w));
    cp_async_commit();
  }
  cp_async_wait<0>();
  __syncthreads();
  const bool pf = threadIdx.x == kHThreads - 32;
  auto slice_prefetch = [&](int t) {
    if (t >= nlev) return;
    const int4 a = ring[0 * kHRing + t % kHRing];
    const int4 b = ring[(kHWarps - 1) * kHRing + t % kHRing];
    if (b.w > a.z) {
      prefetch_l2(lidx + a.z, static_cast<long long>(b.w - a.z) * 4);
      prefetch_l2(lval + a.z, static_cast<long long>(b.w - a.z) * 8);
    }
    if (b.y > a.x) {
      prefetch_l2(lptr + a.x, static_cast<long long>(b.y - a.x + 1) * 8);
      prefetch_l2(rhs_rows + a.x, static_cast<long long>(b.y - a.x) * 8);
      if (FWD) prefetch_l2(dinv_l + a.x, static_cast<long long>(b.y - a.x) * 8);
    }
  };
  if (pf)
    for (int tt = 1; tt <= 4; ++tt) slice_prefetch(tt);
  HeadPre nxt;
  if (nlev > 0) head_load<FWD>(nxt, myring[0], lptr, lidx, lval, rhs_rows, dinv_l, lane);
  // diagnostics (PARAC_SWEEP_PROFILE, cluster): warp 0's per-level phase
  // cycles {load issue, gathers+products, sums+stores, wait+barrier}
  unsigned long long* dbg = (ltime && w == 0 && lane == 0) ? ltime + (FWD ? 20 : 4) * (nlev + 8) : nullptr;
  long long c0 = clock64(), c1 = 0, c2 = 0, c3 = 0;
  for (int t = 0; t < nlev; ++t) {
    if (dbg && t > 0) {
      const long long cn = clock64();
      dbg[4 * (t - 1) + 0] = c1 - c0;
      dbg[4 * (t - 1) + 1] = c2 - c1;
      dbg[4 * (t - 1) + 2] = c3 - c2;
      dbg[4 * (t - 1) + 3] = cn - c3;
      c0 = cn;
    }
    const HeadPre cur = nxt;
    if (t + 1 < nlev) head_load<FWD>(nxt, myring[(t + 1) % kHRing], lptr, lidx, lval, rhs_rows, dinv_l, lane);
    {
      const int tn = t + kHRing - 1;
      if (lane == 0 && tn < nlev) cp_async16(&myring[tn % kHRing], rec_ptr(tn, w));
      cp_async_commit();
    }
    if (pf) slice_prefetch(t + 4);
    if (dbg) c1 = clock64();
    const int jb = cur.rec.x, je = cur.rec.y, eb = cur.rec.z, ee = cur.rec.w;
    const int cnt = ee - eb;
    if (jb < je) {
      if (cnt <= kHeadPF * 32 && je - jb <= 32) {
        // fast path: everything prefetched; one gather round trip
        double xv[kHeadPF];
#pragma unroll
        for (int q = 0; q < kHeadPF; ++q) xv[q] = q * 32 + lane < cnt ? xget(cur.idx[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < kHeadPF; ++q)
          if (q * 32 + lane < cnt) pbuf[q * 32 + lane] = cur.val[q] * xv[q];
        __syncwarp();
        if (dbg) c2 = clock64();
        const int j = jb + lane;
        const int crb = static_cast<int>(cur.rb - eb), cre = static_cast<int>(cur.re - eb);
        const bool mine = j < je && cre - crb <= kShortRow;
        if (mine) {
          double s = 0.0;
          for (int q = crb; q < cre; ++q) s += pbuf[q];
          const double acc = cur.rhs - s;
          xput(j, acc);
          if (FWD) yd_l[j] = acc * cur.dinv;
        }
        unsigned longs = __ballot_sync(kFull, j < je && !mine);
        while (longs) {
          const int src = __ffs(longs) - 1;
          longs &= longs - 1;
          const int b2 = __shfl_sync(kFull, crb, src), e2 = __shfl_sync(kFull, cre, src);
          const double rhs = __shfl_sync(kFull, cur.rhs, src), dv = __shfl_sync(kFull, cur.dinv, src);
          double part = 0.0;
          for (int q = b2 + lane; q < e2; q += 32) part += pbuf[q];
          part = warp_sum(part);
          if (lane == 0) {
            const double acc = rhs - part;
            xput(jb + src, acc);
            if (FWD) yd_l[jb + src] = acc * dv;
          }
        }
        __syncwarp();
      } else if (cnt <= kChunkCap) {
        // many short rows (wide levels): all products first (8 loads in
        // flight per lane), then lane-per-row sums from the product buffer
        for (int base = 0; base < cnt; base += 256) {
          int ci[8];
          double gv[8], xv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int e = base + q * 32 + lane;
            ci[q] = e < cnt ? lidx[eb + e] : 0;
            gv[q] = e < cnt ? lval[eb + e] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) xv[q] = base + q * 32 + lane < cnt ? xget(ci[q]) : 0.0;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (base + q * 32 + lane < cnt) pbuf[base + q * 32 + lane] = gv[q] * xv[q];
        }
        __syncwarp();
        for (int j0 = jb; j0 < je; j0 += 32) {
          const int j = j0 + lane;
          int b = 0, e = 0;
          double rhs = 0.0, dv = 0.0;
          if (j < je) {
            b = static_cast<int>(lptr[j] - eb);
            e = static_cast<int>(lptr[j + 1] - eb);
            rhs = rhs_rows[j];
            if (FWD) dv = dinv_l[j];
          }
          const bool mine = j < je && e - b <= kShortRow;
          if (mine) {
            double sum = 0.0;
            for (int q = b; q < e; ++q) sum += pbuf[q];
            const double acc = rhs - sum;
            xput(j, acc);
            if (FWD) yd_l[j] = acc * dv;
          }
          unsigned longs = __ballot_sync(kFull, j < je && !mine);
          while (longs) {
            const int src = __ffs(longs) - 1;
            longs &= longs - 1;
            const int b2 = __shfl_sync(kFull, b, src), e2 = __shfl_sync(kFull, e, src);
            const double rhs2 = __shfl_sync(kFull, rhs, src), dv2 = __shfl_sync(kFull, dv, src);
            double part = 0.0;
            for (int q = b2 + lane; q < e2; q += 32) part += pbuf[q];
            part = warp_sum(part);
            if (lane == 0) {
              const double acc = rhs2 - part;
              xput(j0 + src, acc);
              if (FWD) yd_l[j0 + src] = acc * dv2;
            }
          }
        }
        __syncwarp();
      } else {
        // general path (wide chunk): rows in batches of 32, products straight from memory
        for (int j0 = jb; j0 < je; j0 += 32) {
          const int j = j0 + lane;
          long long b = 0, e = 0;
          double rhs = 0.0, dv = 0.0;
          if (j < je) {
            b = lptr[j];
            e = lptr[j + 1];
            rhs = rhs_rows[j];
            if (FWD) dv = dinv_l[j];
          }
          if (j < je && e - b <= kShortRow) {
            double s = 0.0;
            for (long long q = b; q < e; ++q) s += lval[q] * xget(lidx[q]);
            const double acc = rhs - s;
            xput(j, acc);
            if (FWD) yd_l[j] = acc * dv;
          }
          unsigned longs = __ballot_sync(kFull, j < je && e - b > kShortRow);
          while (longs) {
            const int src = __ffs(longs) - 1;
            longs &= longs - 1;
            const long long b2 = __shfl_sync(kFull, b, src), e2 = __shfl_sync(kFull, e, src);
            const double rhs2 = __shfl_sync(kFull, rhs, src), dv2 = __shfl_sync(kFull, dv, src);
            double part = 0.0;
            for (long long q = b2 + lane; q < e2; q += 32) part += lval[q] * xget(lidx[q]);
            part = warp_sum(part);
            if (lane == 0) {
              const double acc = rhs2 - part;
              xput(j0 + src, acc);
              if (FWD) yd_l[j0 + src] = acc * dv2;
            }
          }
        }
      }
    }
    if (dbg) c3 = clock64();
    cp_async_wait<2>();  // records of levels <= t + kHRing - 3 have landed
    level_barrier();
    if (ltime && w == 0 && lane == 0) ltime[t] = globaltimer_ns();
  }
  cp_async_wait<0>();
  if constexpr (FWD) {  // tail rows' H part: ts_i = rhs - sum over head columns (idx < tail_base)
    for (int i = w; i < nt; i += W) {
      const int j = tail_base + i;
      const long long b = lptr[j], e = lptr[j + 1];
      double part = 0.0;
      for (long long q = b + lane; q < e; q += 32) {
        const int c = lidx[q];
        if (c < tail_base) part += lval[q] * __ldcg(x + c);
      }
      part = warp_sum(part);
      if (lane == 0) ts[i] = rhs_l[j] - part;
    }
  }
}

// ---- wide levels: one ordinary launch per level. The first ~150 levels of a
// 3D problem hold 10^2-3*10^5 rows of 5-100 entries each: enough independent
// rows to fill the GPU, so the kernel boundary is the level barrier and no
// in-kernel grid barrier is needed. K lanes share a row (K chosen per level
// from its mean row length) so a row's loads issue in parallel; each lane sums
// a fixed stride of the row and the K partials are combined by a fixed xor
// tree (deterministic). Launched with programmatic dependent launch: the
// factor data (row pointers, entries, dinv -- constant during the solve) are
// loaded before griddepcontrol.wait, so the next level's index loads and
// launch overlap the current level; x and the right-hand side are read after.
constexpr int kWideRegs = 4;  // entries per lane staged before the wait

template <bool FWD, int K>
__global__ void __launch_bounds__(256) wide_level_kernel(long long j0, long long j1, const long long* __restrict__ lptr,
                                                          const int* __restrict__ lidx, const double* __restrict__ lval,
                                                          const double* rhs_l, const double* __restrict__ dinv_l,
                                                          double* x, double* yd_l, int rhs_early,
                                                          unsigned long long* lt) {
  const int lane = threadIdx.x % K;
  const long long j = j0 + (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) / K;
  const bool live = j < j1;
  long long b = 0, e = 0;
  if (live) {
    b = lptr[j];
    e = lptr[j + 1];
  }
  int c[kWideRegs];
  double g[kWideRegs];
#pragma unroll
  for (int t = 0; t < kWideRegs; ++t) {
    const long long q = b + lane + static_cast<long long>(t) * K;
    const bool ok = q < e;
    c[t] = ok ? lidx[q] : 0;
    g[t] = ok ? lval[q] : 0.0;
  }
  const bool head = live && lane == 0;
  const double di = (FWD && head) ? dinv_l[j] : 0.0;
  double rh = (rhs_early && head) ? __ldcg(rhs_l + j) : 0.0;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // dependents launch once every CTA of this level is past its wait, i.e. once
  // the level before this one has completed: their early loads never see a
  // vector a kernel still running may write (rhs_early relies on this)
  asm volatile("griddepcontrol.launch_dependents;");
  if (lt && blockIdx.x == 0 && threadIdx.x == 0) *lt = globaltimer_ns();
  double xv[kWideRegs];
#pragma unroll
  for (int t = 0; t < kWideRegs; ++t) xv[t] = __ldcg(x + c[t]);
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < kWideRegs; ++t) s += g[t] * xv[t];
  for (long long q = b + lane + static_cast<long long>(kWideRegs) * K; q < e; q += K) s += lval[q] * __ldcg(x + lidx[q]);
#pragma unroll
  for (int o = K / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (head) {
    if (!rhs_early) rh = __ldcg(rhs_l + j);
    const double acc = rh - s;
    x[j] = acc;
    if (FWD) yd_l[j] = acc * di;
  }
}

template <bool FWD>
cudaError_t launch_wide_level(int K, long long j0, long long j1, cudaStream_t st, const long long* lptr,
                              const int* lidx, const double* lval, const double* rhs_l, const double* dinv_l,
                              double* x, double* yd_l, int rhs_early, unsigned long long* lt) {
  cudaLaunchConfig_t cfg = {};
  const long long threads = (j1 - j0) * K;
  cfg.gridDim = dim3(static_cast<unsigned>((threads + 255) / 256), 1, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
#define PARAC_WIDE_CASE(KK)                                                                                  \
  case KK:                                                                                                   \
    return cudaLaunchKernelEx(&cfg, wide_level_kernel<FWD, KK>, j0, j1, lptr, lidx, lval, rhs_l, dinv_l, x, \
                              yd_l, rhs_early, lt);
  switch (K) {
    PARAC_WIDE_CASE(1)
    PARAC_WIDE_CASE(2)
    PARAC_WIDE_CASE(4)
    PARAC_WIDE_CASE(8)
    PARAC_WIDE_CASE(16)
    default:
      return cudaLaunchKernelEx(&cfg, wide_level_kernel<FWD, 32>, j0, j1, lptr, lidx, lval, rhs_l, dinv_l, x, yd_l,
                                rhs_early, lt);
  }
#undef PARAC_WIDE_CASE
}

// lanes per row for a level of `rows` rows and `ents` entries: the mean row
// spread over <= kWideRegs entries per lane, at most a warp
inline int wide_lanes(long long rows, long long ents) {
  const long long mean = rows > 0 ? (ents + rows - 1) / rows : 1;
  int K = 1;
  while (K < 32 && static_cast<long long>(K) * kWideRegs < mean) K *= 2;
  return K;
}

__global__ void rhs_permute_kernel(int n, const int* rlab, const double* r, double* rhs_l) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) rhs_l[j] = r[rlab[j]];
}

// hrec[L][w]: chunk w of level L (whole rows, ~equal entries + rows), for W warps.
__global__ void head_chunk_kernel(int depth, int W, const long long* lvl_off, const long long* lptr, int4* hrec) {
  const int L = blockIdx.x + 1;
  if (L > depth) return;
  const long long lb = lvl_off[L], le = lvl_off[L + 1];
  const long long tot = (lptr[le] - lptr[lb]) + (le - lb);
  auto start = [&](int c) -> long long {
    if (c >= W) return le;
    const long long goal = (tot * c + W - 1) / W;
    long long lo = lb, hi = le;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if ((lptr[mid] - lptr[lb]) + (mid - lb) >= goal) hi = mid; else lo = mid + 1;
    }
    return lo;
  };
  for (int c = threadIdx.x; c < W; c += blockDim.x) {
    const long long a = start(c), b = start(c + 1);
    hrec[static_cast<long long>(L) * W + c] =
        make_int4(static_cast<int>(a), static_cast<int>(b), static_cast<int>(lptr[a]), static_cast<int>(lptr[b]));
  }
}

// Level-order remaps: lpos[order[j]] = j; rlab[j] = inv[order[j]];
// dinv_l[j] = D^+ of row order[j]; v2l[label] = lpos[perm[label]].
__global__ void level_maps_kernel(int n, const int* order, const int* inv, const double* diag, int* lpos,
                                  int* rlab, double* dinv_l) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int r = order[j];
  lpos[r] = j;
  rlab[j] = inv[r];
  const double d = diag[r];
  dinv_l[j] = d > 0.0 ? 1.0 / d : 0.0;
}
__global__ void label_map_kernel(int n, const int* perm, const int* lpos, int* v2l) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) v2l[v] = lpos[perm[v]];
}
__global__ void remap_idx_kernel(long long cnt, const int* lpos, int* idx) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < cnt;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    idx[e] = lpos[idx[e]];
}
__global__ void gather_z_l_dot_kernel(int n, const int* v2l, const double* zl, const double* r, double* z,
                                      double* partials) {
  double s = 0.0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const double zv = zl[v2l[v]];
    z[v] = zv;
    s += r[v] * zv;
  }
  block_partial(s, partials);
}

#include "tail_dense.cuh"

// T-part of the forward tail rows: count, then copy with tail-relative indices.
__global__ void tail3_count_kernel(int nt, int tail_base, const long long* lptr, const int* lidx, int* cnt) {
  const int lane = lane_id();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < nt; i += nw) {
    const long long b = lptr[tail_base + i], e = lptr[tail_base + i + 1];
    int c = 0;
    for (long long q = b + lane; q < e; q += 32) c += lidx[q] >= tail_base;
    c = warp_sum(c);
    if (lane == 0) cnt[i] = c;
  }
}
__global__ void tail3_fill_kernel(int nt, int tail_base, const long long* lptr, const int* lidx, const double* lval,
                                  const long long* off, int* tidx, double* tval) {
  const int lane = lane_id();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < nt; i += nw) {
    const long long b = lptr[tail_base + i], e = lptr[tail_base + i + 1];
    long long o = off[i];
    for (long long q0 = b; q0 < e; q0 += 32) {
      const long long q = q0 + lane;
      const bool t = q < e && lidx[q] >= tail_base;
      const unsigned m = __ballot_sync(kFull, t);
      if (t) {
        const long long at = o + __popc(m & ((1u << lane) - 1));
        tidx[at] = lidx[q] - tail_base;
        tval[at] = lval[q];
      }
      o += __popc(m);
    }
  }
}
__global__ void ll_to_int_kernel(int cnt, const long long* src, long long base, int* dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) dst[i] = static_cast<int>(src[i] - base);
}
// Level-ordered row copies: lens, then entries (warp per row).
__global__ void lvl_len_kernel(int n, const int* order, const long long* aptr, const long long* bptr,
                               int* alen, int* blen) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int r = order[j];
  alen[j] = static_cast<int>(aptr[r + 1] - aptr[r]);
  blen[j] = static_cast<int>(bptr[r + 1] - bptr[r]);
}

__global__ void lvl_copy_kernel(int n, const int* order, const long long* src_ptr, const int* src_idx,
                                const double* src_val, const long long* dst_ptr, int* dst_idx, double* dst_val) {
  const int lane = lane_id();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int j = gw; j < n; j += nw) {
    const int r = order[j];
    const long long sb = src_ptr[r], se = src_ptr[r + 1], db = dst_ptr[j];
    for (long long q = sb + lane; q < se; q += 32) {
      dst_idx[db + (q - sb)] = src_idx[q];
      dst_val[db + (q - sb)] = src_val[q];
    }
  }
}


template <typename... KArgs, typename... Args>
cudaError_t launch_cluster_t(void (*kernel)(KArgs...), int csize, int threads, std::size_t smem, cudaStream_t st,
                             Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_cluster(void (*kernel)(KArgs...), int csize, std::size_t smem, cudaStream_t st, Args... args) {
  return launch_cluster_t(kernel, csize, kCThreads, smem, st, args...);
}


// Ordinary launch with programmatic dependent launch enabled (the kernel calls
// griddepcontrol.wait before reading its predecessor's output).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int threads, std::size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid), 1, 1);
  cfg.blockDim = dim3(static_cast<unsigned>(threads), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Largest launchable cluster (16 non-portable, else 8) of 1024-thread CTAs.
template <typename... KArgs>
int pick_cluster(void (*kernel)(KArgs...), std::size_t smem = 0, int threads = kCThreads) {
  if (smem) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  for (int c : {16, 8, 4}) {
    if (c > 8) cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c, 1, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kernel, &cfg) == cudaSuccess && nclusters > 0) return c;
    cudaGetLastError();
  }
  return 1;
}

struct ClusterSizes {
  int fwd_exact, bwd_exact;
};
ClusterSizes cluster_sizes(int device) {
  static ClusterSizes cached[64] = {};
  if (device >= 0 && device < 64 && cached[device].fwd_exact) return cached[device];
  ClusterSizes c{pick_cluster(cluster_forward_kernel<true>), pick_cluster(cluster_backward_kernel<true>)};
  if (device >= 0 && device < 64) cached[device] = c;
  return c;
}

// Grid of the sync-free level pass (uploaded factors): exactly its co-resident
// capacity, so every CTA that a waiting row depends on is resident.
int sweep_grid(int device) {
  static int cached[64] = {};
  if (device >= 0 && device < 64 && cached[device]) return cached[device];
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, level_kernel, kSweepThreads, 0);
  const int g = std::max(1, per_sm) * sm_count(device);
  if (device >= 0 && device < 64) cached[device] = g;
  return g;
}

// ---------------------------------------------------------------- host side
void drop_pcg_graph(SolveState& s) {
  if (s.pcg_exec) cudaGraphExecDestroy(s.pcg_exec);
  if (s.pcg_graph) cudaGraphDestroy(s.pcg_graph);
  s.pcg_exec = nullptr;
  s.pcg_graph = nullptr;
}

void ensure_vectors(SolveState& s, int n) {
  if (s.cap_n >= static_cast<std::size_t>(n) && s.x) return;
  drop_pcg_graph(s);  // its kernels hold the old vectors
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
  if (s.graph_ready && s.components >= 0) return s.components;  // once per staged graph
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
  s.components = h;
  return h;
}


__global__ void gather_ll_kernel(int cnt, const long long* idx, const long long* src, long long* dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) dst[i] = src[idx[i]];
}


// Level-ordered copies of G's rows and columns + chunk tables (fast mode).
void build_level_layout(const SolveInputs& in, SolveState& s, int sms) {
  const int n = in.f_n, depth = s.depth;
  const long long Z = in.f_nnz;
  cudaStream_t st = in.stream;
  if (n == 0 || depth == 0) return;
  const std::size_t cz = static_cast<std::size_t>(std::max<long long>(Z, 1));
  if (s.cap_lz < cz) {
    dalloc(s.lf_idx, cz); dalloc(s.lf_val, cz); dalloc(s.lb_idx, cz); dalloc(s.lb_val, cz);
    s.cap_lz = cz;
  }
  if (s.cap_levels < static_cast<std::size_t>(n) + 2) {
    dalloc(s.lf_ptr, static_cast<std::size_t>(n) + 1);
    dalloc(s.lb_ptr, static_cast<std::size_t>(n) + 1);
    dalloc(s.lvl_target, static_cast<std::size_t>(n) + 2);
    s.cap_levels = static_cast<std::size_t>(n) + 2;
  }
  int* alen = s.tmp_int;
  int* blen = nullptr;
  dalloc(blen, static_cast<std::size_t>(n) + 1);
  const int blocks = (n + 255) / 256;
  lvl_len_kernel<<<blocks, 256, 0, st>>>(n, s.order, s.gt_ptr, in.col_ptr, alen, blen);
  note_launches(1);
  check(launch_scan(alen, n, s.lf_ptr, s.tiles, st), "scan");
  check(launch_scan(blen, n, s.lb_ptr, s.tiles, st), "scan");
  lvl_copy_kernel<<<sms * 8, 256, 0, st>>>(n, s.order, s.gt_ptr, s.gt_col, s.gt_val, s.lf_ptr, s.lf_idx, s.lf_val);
  lvl_copy_kernel<<<sms * 8, 256, 0, st>>>(n, s.order, in.col_ptr, in.rows, in.vals, s.lb_ptr, s.lb_idx, s.lb_val);
  note_launches(2);
  dfree(blen);
  check(cudaGetLastError(), "level layout");
}

// v3 fast-mode layout (after build_level_layout made the level-ordered copies):
// level-order maps, indices remapped to level order, head chunk tables for the
// cluster's warps, and the dense-inverse tail (tail_dense.cuh).
void build_fast_v3(const SolveInputs& in, SolveState& s, int sms) {
  const int n = in.f_n, depth = s.depth;
  const long long Z = in.f_nnz;
  cudaStream_t st = in.stream;
  s.t3_L0 = depth;
  s.t3_nt = 0;
  s.t3_base = n;
  s.t3_nlev = 0;
  if (n == 0 || depth == 0) return;
  const std::size_t nn = static_cast<std::size_t>(n);
  if (s.cap_v3 < nn) {
    dalloc(s.lpos, nn); dalloc(s.rlab, nn); dalloc(s.v2l, nn); dalloc(s.dinv_l, nn); dalloc(s.rhs_l, nn);
    s.cap_v3 = nn;
  }
  const int blocks = (n + 255) / 256;
  level_maps_kernel<<<blocks, 256, 0, st>>>(n, s.order, s.inv, in.diag, s.lpos, s.rlab, s.dinv_l);
  label_map_kernel<<<blocks, 256, 0, st>>>(n, in.perm, s.lpos, s.v2l);
  remap_idx_kernel<<<sms * 8, 256, 0, st>>>(Z, s.lpos, s.lf_idx);
  remap_idx_kernel<<<sms * 8, 256, 0, st>>>(Z, s.lpos, s.lb_idx);
  note_launches(4);
  // head cluster geometry + chunk tables (all levels; the head uses 1..L0)
  static int csize[64] = {};
  const int dev = in.device >= 0 && in.device < 64 ? in.device : 0;
  if (!csize[dev]) {
    csize[dev] = pick_cluster(head_sweep_kernel<true>, kHeadSmem, kHThreads);
    if (const char* hc = std::getenv("PARAC_HEAD_CLUSTER"))  // tuning: a smaller head cluster (1..16)
      csize[dev] = std::max(1, std::min(csize[dev], std::atoi(hc)));
    cudaFuncSetAttribute(head_sweep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kHeadSmem));
    cudaFuncSetAttribute(head_sweep_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  s.head_csize = csize[dev];
  s.head_W = s.head_csize * kHWarps;
  const std::size_t nrec = (static_cast<std::size_t>(depth) + 2) * s.head_W;
  if (s.cap_hrec < nrec) {
    dalloc(s.hrec_f, nrec);
    dalloc(s.hrec_b, nrec);
    s.cap_hrec = nrec;
  }
  head_chunk_kernel<<<depth, 256, 0, st>>>(depth, s.head_W, s.lvl_off, s.lf_ptr, s.hrec_f);
  head_chunk_kernel<<<depth, 256, 0, st>>>(depth, s.head_W, s.lvl_off, s.lb_ptr, s.hrec_b);
  note_launches(2);
  // tail choice
  std::vector<long long> off(static_cast<std::size_t>(depth) + 2);
  check(cudaMemcpyAsync(off.data(), s.lvl_off, sizeof(long long) * (depth + 2), cudaMemcpyDeviceToHost, st), "d2h");
  check(cudaStreamSynchronize(st), "v3 sync");
  // wide leading levels (one launch per level): rows + entries (forward rows
  // and backward columns) above PARAC_WIDE_WEIGHT (default 16384)
  {
    const char* ww = std::getenv("PARAC_WIDE_WEIGHT");
    const long long wide = ww ? std::atoll(ww) : 16384;
    std::vector<long long> ef(static_cast<std::size_t>(depth) + 2), eb(static_cast<std::size_t>(depth) + 2);
    long long* bnd = s.lvl_target;
    gather_ll_kernel<<<(depth + 2 + 255) / 256, 256, 0, st>>>(depth + 2, s.lvl_off, s.lf_ptr, bnd);
    check(cudaMemcpyAsync(ef.data(), bnd, sizeof(long long) * (depth + 2), cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaStreamSynchronize(st), "v3 sync");
    gather_ll_kernel<<<(depth + 2 + 255) / 256, 256, 0, st>>>(depth + 2, s.lvl_off, s.lb_ptr, bnd);
    check(cudaMemcpyAsync(eb.data(), bnd, sizeof(long long) * (depth + 2), cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaStreamSynchronize(st), "v3 sync");
    note_launches(2);
    int Lw = 0;
    while (Lw < depth) {
      const int L = Lw + 1;
      const long long rows = off[L + 1] - off[L];
      const long long wgt = rows + std::max(ef[L + 1] - ef[L], eb[L + 1] - eb[L]);
      if (wide <= 0 || wgt < wide) break;
      Lw = L;
    }
    s.wide_L = Lw;
    s.wide_kf.assign(static_cast<std::size_t>(Lw) + 1, 1);
    s.wide_kb.assign(static_cast<std::size_t>(Lw) + 1, 1);
    for (int L = 1; L <= Lw; ++L) {
      s.wide_kf[L] = wide_lanes(off[L + 1] - off[L], ef[L + 1] - ef[L]);
      s.wide_kb[L] = wide_lanes(off[L + 1] - off[L], eb[L + 1] - eb[L]);
    }
    s.lvl_off_h.assign(off.begin(), off.begin() + std::min<std::size_t>(off.size(), static_cast<std::size_t>(Lw) + 2));
  }
  // Dense-inverse tail (tail_dense.cuh): the trailing levels whose rows fit
  // T <= kTwMaxRows. Which levels: the split minimising a cost model of the
  // per-apply time (2 GEMVs of T^2/2 x 8 bytes vs one cluster-barrier level
  // per head level and direction) amortised over ~40 applies plus the one-time
  // build (~T-weighted entry count x 8 bytes + one launch per tail level).
  // PARAC_TAIL_ROWS=T forces the largest tail of at most T rows (0: none).
  const int Lw = s.wide_L;
  int L0 = depth;  // last head level; the tail is levels L0+1 .. depth
  {
    const char* env = std::getenv("PARAC_TAIL_ROWS");
    const long long forced = env ? std::atoll(env) : -1;
    const long long cap = std::min<long long>(forced >= 0 ? forced : kTwMaxRows, kTwMaxRows);
    std::vector<long long> ef(static_cast<std::size_t>(depth) + 2);
    gather_ll_kernel<<<(depth + 2 + 255) / 256, 256, 0, st>>>(depth + 2, s.lvl_off, s.lf_ptr, s.lvl_target);
    note_launches(1);
    check(cudaMemcpyAsync(ef.data(), s.lvl_target, sizeof(long long) * (depth + 2), cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaStreamSynchronize(st), "v3 sync");
    constexpr double kGemvBW = 5.0e12, kBuildBW = 2.5e12, kHeadLevel = 2.8e-6, kLaunch = 4.0e-6, kApplies = 40.0;
    double best = 1e300;
    double S0 = 0.0, S1 = 0.0;  // sums over tail levels l of E_l and E_l * off[l]
    for (int Lc = depth; Lc >= std::max(Lw, 0); --Lc) {  // candidate: tail = levels Lc+1 .. depth
      const long long tb = off[Lc + 1], T = n - tb;
      if (T > cap) break;
      if (Lc < depth) {
        const double El = static_cast<double>(ef[Lc + 2] - ef[Lc + 1]);
        S0 += El;
        S1 += El * static_cast<double>(off[Lc + 1]);
      }
      // build traffic: each tail entry of level l reads a parent row of mean
      // length ~ (tail-relative start of level l) / 2
      const double fma_bytes = 0.5 * (S1 - static_cast<double>(tb) * S0) * 8.0;
      const double Td = static_cast<double>(T);
      const double apply = 2.0 * (Td * Td * 4.0 / kGemvBW + (T ? 3e-6 : 0.0)) + 2.0 * kHeadLevel * (Lc - Lw);
      const double cost = apply * kApplies + fma_bytes / kBuildBW + (depth - Lc) * kLaunch;
      if (forced >= 0 || cost < best) {
        best = cost;
        L0 = Lc;
      }
    }
  }
  s.t3_L0 = L0;
  if (L0 >= depth) return;
  const int base = static_cast<int>(off[L0 + 1]);
  const int nt = n - base;
  const int nlev = depth - L0;
  const int Tp = tw_even(nt);
  if (s.cap_t3 < static_cast<std::size_t>(nt) + 2) {
    dalloc(s.t3_fep, static_cast<std::size_t>(nt) + 2);
    dalloc(s.tail_s, static_cast<std::size_t>(nt) + 2);
    dalloc(s.tail_cnt, 2 * (static_cast<std::size_t>(nt) + 2));
    dalloc(s.hsplit, static_cast<std::size_t>(nt) + 2);  // scratch: forward T-part offsets
    dalloc(s.tw_offl, static_cast<std::size_t>(nt) + 2);
    dalloc(s.tw_offu, static_cast<std::size_t>(nt) + 2);
    s.cap_t3 = static_cast<std::size_t>(nt) + 2;
  }
  // forward T part of every tail row (entries with tail-relative indices)
  tail3_count_kernel<<<sms * 4, 256, 0, st>>>(nt, base, s.lf_ptr, s.lf_idx, s.tail_cnt);
  note_launches(1);
  check(launch_scan(s.tail_cnt, nt, s.hsplit, s.tiles, st), "scan");
  long long hb = 0;
  check(cudaMemcpyAsync(&hb, s.hsplit + nt, sizeof(long long), cudaMemcpyDeviceToHost, st), "d2h");
  check(cudaStreamSynchronize(st), "v3 sync");
  const std::size_t ne = static_cast<std::size_t>(std::max<long long>(hb, 1));
  if (s.cap_t3e < ne) {
    dalloc(s.t3_fidx, ne);
    dalloc(s.t3_fval, ne);
    s.cap_t3e = ne;
  }
  tail3_fill_kernel<<<sms * 4, 256, 0, st>>>(nt, base, s.lf_ptr, s.lf_idx, s.lf_val, s.hsplit, s.t3_fidx, s.t3_fval);
  ll_to_int_kernel<<<(nt + 1 + 255) / 256, 256, 0, st>>>(nt + 1, s.hsplit, 0, s.t3_fep);
  note_launches(2);
  // packed row offsets of W (lower) and W^T (upper), padded to even lengths
  std::vector<long long> offl(static_cast<std::size_t>(nt) + 1), offu(static_cast<std::size_t>(nt) + 1);
  offl[0] = offu[0] = 0;
  for (int i = 0; i < nt; ++i) {
    offl[i + 1] = offl[i] + tw_even(i + 1);
    offu[i + 1] = offu[i] + (Tp - (i & ~1));
  }
  check(cudaMemcpyAsync(s.tw_offl, offl.data(), sizeof(long long) * (nt + 1), cudaMemcpyHostToDevice, st), "h2d");
  check(cudaMemcpyAsync(s.tw_offu, offu.data(), sizeof(long long) * (nt + 1), cudaMemcpyHostToDevice, st), "h2d");
  const std::size_t wl = static_cast<std::size_t>(offl[nt]), wu = static_cast<std::size_t>(offu[nt]);
  if (s.cap_tw < wl || s.cap_twt < wu) {
    dalloc(s.tw, std::max(wl, s.cap_tw));
    dalloc(s.twt, std::max(wu, s.cap_twt));
    s.cap_tw = std::max(wl, s.cap_tw);
    s.cap_twt = std::max(wu, s.cap_twt);
  }
  // W = G_TT^-1, one launch per tail level (programmatic dependent launch:
  // the next level's entries are staged while this one finishes)
  for (int t = 0; t < nlev; ++t) {
    const int r0 = static_cast<int>(off[L0 + 1 + t] - base), r1 = static_cast<int>(off[L0 + 2 + t] - base);
    if (r1 <= r0) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>((tw_even(r1) + kTwBlockCols - 1) / kTwBlockCols),
                       static_cast<unsigned>(r1 - r0), 1);
    cfg.blockDim = dim3(kTwBuildThreads, 1, 1);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    check(cudaLaunchKernelEx(&cfg, tw_build_level_kernel, r0, r1, static_cast<const int*>(s.t3_fep),
                             static_cast<const int*>(s.t3_fidx), static_cast<const double*>(s.t3_fval),
                             static_cast<const long long*>(s.tw_offl), s.tw),
          "tail W build");
    note_launches(1);
  }
  {
    const long long nb = (Tp + 31) / 32;
    tw_transpose_kernel<<<static_cast<unsigned>(nb * (nb + 1) / 2), 256, 0, st>>>(nt, Tp, s.tw, s.tw_offl, s.tw_offu,
                                                                                  s.twt);
    note_launches(1);
  }
  // kernel attributes belong to each device's context: set them per device
  static bool attr[64] = {};
  if (!attr[dev]) {
    const int smem = static_cast<int>(sizeof(double) * kTwMaxRows);
    check(cudaFuncSetAttribute(tw_gemv_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "attr");
    check(cudaFuncSetAttribute(tw_gemv_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "attr");
    attr[dev] = true;
  }
  check(cudaGetLastError(), "v3 layout");
  s.t3_nt = nt;
  s.t3_base = base;
  s.t3_nlev = nlev;
  s.tw_T = nt;
  s.tw_Tp = Tp;
}

void prepare_factor(const SolveInputs& in) {
  SolveState& s = *in.state;
  if (s.factor_ready) return;
  drop_pcg_graph(s);  // captured for the previous factor's layout
  const int n = in.f_n;
  const long long Z = in.f_nnz;
  cudaStream_t st = in.stream;
  const int blocks = (n + 255) / 256;
  const int sms = sm_count(in.device);
  static const bool verbose = std::getenv("PARAC_VERBOSE") != nullptr;
  auto t_start = std::chrono::steady_clock::now();
  auto stamp = [&](const char* what) {
    if (!verbose) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "prepare_factor %-16s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_start).count());
    t_start = now;
  };
  if (s.cap_z < static_cast<std::size_t>(std::max<long long>(Z, 1))) {
    const std::size_t cz = static_cast<std::size_t>(std::max<long long>(Z, 1));
    dalloc(s.gt_col, cz);
    dalloc(s.gt_val, cz);
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
  {  // rows longer than kGtShortRow
    int* flag = s.tmp_int;
    int* len = nullptr;
    long long* rpos = nullptr;
    long long* loff = nullptr;
    check(cudaMallocAsync(&len, sizeof(int) * (static_cast<std::size_t>(n) + 1), st), "alloc");
    check(cudaMallocAsync(&rpos, sizeof(long long) * (static_cast<std::size_t>(n) + 1), st), "alloc");
    check(cudaMallocAsync(&loff, sizeof(long long) * (static_cast<std::size_t>(n) + 1), st), "alloc");
    gt_long_flags_kernel<<<blocks, 256, 0, st>>>(n, s.gt_ptr, flag, len);
    note_launches(1);
    check(launch_scan(flag, n, rpos, s.tiles, st), "scan");
    check(launch_scan(len, n, loff, s.tiles, st), "scan");
    long long tot[2] = {0, 0};
    check(cudaMemcpyAsync(&tot[0], rpos + n, sizeof(long long), cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaMemcpyAsync(&tot[1], loff + n, sizeof(long long), cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaStreamSynchronize(st), "long rows");
    const int nl = static_cast<int>(tot[0]);
    const long long T = tot[1];
    if (nl > 0) {
      int *beg, *end, *rows, *ck, *ck2;
      double *cv, *cv2;
      check(cudaMallocAsync(&beg, sizeof(int) * nl, st), "alloc");
      check(cudaMallocAsync(&end, sizeof(int) * nl, st), "alloc");
      check(cudaMallocAsync(&rows, sizeof(int) * nl, st), "alloc");
      check(cudaMallocAsync(&ck, sizeof(int) * T, st), "alloc");
      check(cudaMallocAsync(&ck2, sizeof(int) * T, st), "alloc");
      check(cudaMallocAsync(&cv, sizeof(double) * T, st), "alloc");
      check(cudaMallocAsync(&cv2, sizeof(double) * T, st), "alloc");
      gt_long_gather_kernel<<<sms * 8, 256, 0, st>>>(n, s.gt_ptr, flag, rpos, loff, s.gt_col, s.gt_val, beg, end,
                                                     rows, ck, cv);
      int cb = 1;
      while (cb < 31 && (1LL << cb) < n) ++cb;
      int sb = 1;
      while (sb < 31 && (1LL << sb) < nl) ++sb;
      unsigned long long *ka, *kb2;
      int *ia, *ib;
      check(cudaMallocAsync(&ka, sizeof(unsigned long long) * T, st), "alloc");
      check(cudaMallocAsync(&kb2, sizeof(unsigned long long) * T, st), "alloc");
      check(cudaMallocAsync(&ia, sizeof(int) * T, st), "alloc");
      check(cudaMallocAsync(&ib, sizeof(int) * T, st), "alloc");
      gt_long_keys_kernel<<<std::min(nl, sms * 8), 256, 0, st>>>(nl, beg, end, ck, cb, ka, ia);
      note_launches(1);
      unsigned long long* kk[2] = {ka, kb2};
      int* ii[2] = {ia, ib};
      const int cur = radix::sort_pairs(static_cast<int>(T), kk, ii, cb + sb, st);
      gt_long_unkey_kernel<<<sms * 8, 256, 0, st>>>(T, kk[cur], ii[cur], (1ULL << cb) - 1, cv, ck2, cv2);
      note_launches(1);
      for (void* q : {static_cast<void*>(ka), static_cast<void*>(kb2), static_cast<void*>(ia), static_cast<void*>(ib)})
        check(cudaFreeAsync(q, st), "free");
      gt_long_scatter_kernel<<<sms * 8, 256, 0, st>>>(nl, s.gt_ptr, beg, end, rows, ck2, cv2, s.gt_col, s.gt_val);
      note_launches(2);
      for (void* q : {static_cast<void*>(beg), static_cast<void*>(end), static_cast<void*>(rows),
                      static_cast<void*>(ck), static_cast<void*>(ck2), static_cast<void*>(cv),
                      static_cast<void*>(cv2)})
        check(cudaFreeAsync(q, st), "free");
    }
    check(cudaFreeAsync(rpos, st), "free");
    check(cudaFreeAsync(loff, st), "free");
    check(cudaFreeAsync(len, st), "free");
  }
  stamp("transpose");
  // levels: recorded by the elimination kernel for factors computed here,
  // recomputed (sync-free pass over G's rows) for uploaded ones
  check(cudaMemsetAsync(s.counters, 0, sizeof(int) * 4, st), "memset");
  if (in.level) {
    check(cudaMemcpyAsync(s.level, in.level, sizeof(int) * n, cudaMemcpyDeviceToDevice, st), "d2d");
  } else {
    const int stamp = ++s.epoch;
    level_kernel<<<sweep_grid(in.device), kSweepThreads, 0, st>>>(n, s.gt_ptr, s.gt_col, s.level,
                                                                  s.flags, stamp, s.counters, s.counters + 3);
    note_launches(1);
    int abort_flag = 0;
    check(cudaMemcpyAsync(&abort_flag, s.counters + 3, sizeof(int), cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaStreamSynchronize(st), "levels");
    if (abort_flag) throw Failure{dimension_mismatch, "factor is not lower triangular (level analysis aborted)"};
  }
  // counting sort of positions by level
  int* hist = s.tmp_int;  // levels are 1..n
  check(cudaMemsetAsync(hist, 0, sizeof(int) * (n + 2), st), "memset");
  level_hist_kernel<<<blocks, 256, 0, st>>>(n, s.level, hist, s.counters + 1);
  note_launches(2);
  check(launch_scan(hist, n + 1, s.lvl_off, s.tiles, st), "scan");
  int depth = 0;
  check(cudaMemcpyAsync(&depth, s.counters + 1, sizeof(int), cudaMemcpyDeviceToHost, st), "d2h");
  check(cudaStreamSynchronize(st), "prepare_factor");
  s.depth = depth;
  // positions in (level, position) order: a STABLE sort by level, so the
  // level-order layout -- and with it every fast-mode summation order -- is
  // the same on every build of the same factor (an atomic scatter was not)
  {
    int* key_a = nullptr;
    int* key_b = nullptr;
    int* pos_in = nullptr;
    const std::size_t nb = sizeof(int) * static_cast<std::size_t>(std::max(n, 1));
    check(cudaMallocAsync(&key_a, nb, st), "alloc");
    check(cudaMallocAsync(&key_b, nb, st), "alloc");
    check(cudaMallocAsync(&pos_in, nb, st), "alloc");
    check(cudaMemcpyAsync(key_a, s.level, sizeof(int) * static_cast<std::size_t>(n), cudaMemcpyDeviceToDevice, st),
          "level copy");
    iota_kernel<<<blocks, 256, 0, st>>>(n, pos_in);
    note_launches(1);
    int bits = 1;
    while (bits < 31 && (1 << bits) <= depth) ++bits;
    int* kb[2] = {key_a, key_b};
    int* vb[2] = {pos_in, s.order};
    const int cur = radix::sort_pairs(n, kb, vb, bits, st);
    if (vb[cur] != s.order)
      check(cudaMemcpyAsync(s.order, vb[cur], sizeof(int) * static_cast<std::size_t>(n), cudaMemcpyDeviceToDevice, st),
            "order copy");
    for (void* q : {static_cast<void*>(key_a), static_cast<void*>(key_b), static_cast<void*>(pos_in)})
      check(cudaFreeAsync(q, st), "free");
  }
  stamp("levels");
  build_level_layout(in, s, sms);
  stamp("level layout");
  build_fast_v3(in, s, sms);
  stamp("v3 tables");
  if (std::getenv("PARAC_SWEEP_PROFILE")) {
    const std::size_t need = 16 * (static_cast<std::size_t>(s.depth) + 2);
    if (s.cap_ltime < need) {
      dalloc(s.ltime, need);
      s.cap_ltime = need;
    }
    check(cudaMemsetAsync(s.ltime, 0, need * 8, st), "memset");
  }
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
  std::vector<double> hp = std::vector<double>(kRedBlocks);

  explicit Solver(const SolveInputs& i)
      : in(i), s(*i.state), st(i.stream), n(i.n) {}

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
    if (!exact) {
      const int H = s.t3_L0, nt = s.t3_nt;
      const int Lw = std::min(s.wide_L, H);
      unsigned long long* lt = s.ltime;
      // forward: rhs into level order, wide levels (one launch each), cluster head, tail
      rhs_permute_kernel<<<(in.f_n + 255) / 256, 256, 0, st>>>(in.f_n, s.rlab, r, s.rhs_l);
      note_launches(1);
      for (int L = 1; L <= Lw; ++L) {
        const long long j0 = s.lvl_off_h[L], j1 = s.lvl_off_h[L + 1];
        check(launch_wide_level<true>(s.wide_kf[L], j0, j1, st, s.lf_ptr, s.lf_idx, s.lf_val, s.rhs_l, s.dinv_l,
                                      s.yf, s.yd, L >= 2, lt ? lt + (L - 1) : nullptr), "wide level forward");
      }
      note_launches(Lw);
      if (H > Lw) {
        check(launch_cluster_t(head_sweep_kernel<true>, s.head_csize, kHThreads, kHeadSmem, st, Lw + 1, H - Lw,
                               s.head_W, s.hrec_f, s.lf_ptr, s.lf_idx, s.lf_val, s.rhs_l, s.dinv_l, s.yf, s.yd, 0,
                               s.t3_base, s.tail_s, lt ? lt + Lw : nullptr),
              "head forward");
        note_launches(1);
      }
      // dense-inverse tail: ts = rhs_T - G_TH y_H, then y_T = W ts (+ D^+),
      // z_T = W^T (D^+ y)_T (tail_dense.cuh)
      if (nt > 0) {
        const int base = s.t3_base;
        tail_rhs_kernel<<<sm_count(in.device) * 4, 256, 0, st>>>(nt, base, s.lf_ptr, s.lf_idx, s.lf_val, s.rhs_l,
                                                                s.yf, s.tail_s);
        note_launches(1);
        const std::size_t smem = sizeof(double) * static_cast<std::size_t>(s.tw_Tp);
        check(launch_pdl(tw_gemv_kernel<true>, sm_count(in.device), kTwGemvThreads, smem, st, nt, s.tw_Tp,
                         static_cast<const double*>(s.tw), static_cast<const long long*>(s.tw_offl),
                         static_cast<const double*>(s.tail_s), static_cast<const double*>(s.dinv_l + base),
                         s.yf + base, s.yd + base),
              "tail forward");
        check(launch_pdl(tw_gemv_kernel<false>, sm_count(in.device), kTwGemvThreads, smem, st, nt, s.tw_Tp,
                         static_cast<const double*>(s.twt), static_cast<const long long*>(s.tw_offu),
                         static_cast<const double*>(s.yd + base), static_cast<const double*>(nullptr), s.zb + base,
                         static_cast<double*>(nullptr)),
              "tail backward");
        note_launches(2);
      }
      // backward: cluster head, wide levels
      if (H > Lw) {
        check(launch_cluster_t(head_sweep_kernel<false>, s.head_csize, kHThreads, kHeadSmem, st, H, H - Lw,
                               s.head_W, s.hrec_b, s.lb_ptr, s.lb_idx, s.lb_val, s.yd, nullptr, s.zb, nullptr, 0, 0,
                               nullptr, lt ? lt + 3 * (D + 2) : nullptr),
              "head backward");
        note_launches(1);
      }
      for (int L = Lw; L >= 1; --L) {
        const long long j0 = s.lvl_off_h[L], j1 = s.lvl_off_h[L + 1];
        check(launch_wide_level<false>(s.wide_kb[L], j0, j1, st, s.lb_ptr, s.lb_idx, s.lb_val, s.yd, nullptr, s.zb,
                                       nullptr, 1, lt ? lt + 3 * (D + 2) + (H - Lw) + (Lw - L) : nullptr),
              "wide level backward");
      }
      note_launches(Lw);
      gather_z_l_dot_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(in.f_n, s.v2l, s.zb, r, z, part(slot));
      note_launches(2);
      return;
    }
    // exact mode: bit-identical to apply_preconditioner (serial row sums in the
    // reference's order), one cluster per direction over all levels
    const ClusterSizes cs = cluster_sizes(in.device);
    check(launch_cluster(cluster_forward_kernel<true>, cs.fwd_exact, 0, st, D, s.lvl_off, s.order, s.gt_ptr,
                         s.gt_col, s.gt_val, in.diag, s.inv, r, s.yf, s.yd, 0, 0, nullptr, nullptr, nullptr,
                         nullptr), "cluster forward");
    check(launch_cluster(cluster_backward_kernel<true>, cs.bwd_exact, 0, st, D, s.lvl_off, s.order, in.col_ptr,
                         in.rows, in.vals, s.yd, s.zb), "cluster backward");
    gather_z_dot_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(in.f_n, in.perm, s.zb, r, z, part(slot));
    note_launches(3);
  }

  void spmv(const double* x, double* y, int slot) {
    spmv_dot_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, in.ptr, in.adj, in.w, s.wdeg, x, y, part(slot));
    note_launches(1);
  }

  // Serial chain(s) in the reference's order (exact PCG); blocking read.
  void chains(Chain c0, Chain c1, int nch, double* out) {
    serial_chain_kernel<<<1, kSerThreads, 0, st>>>(n, c0, c1, nch, s.scalars + 4);
    note_launches(1);
    check(cudaMemcpyAsync(out, s.scalars + 4, sizeof(double) * nch, cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaStreamSynchronize(st), "sync");
  }
  double chain(int kind, const double* a, const double* b = nullptr) {
    double v = 0.0;
    chains(Chain{kind, a, b}, Chain{kind, a, b}, 1, &v);
    return v;
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
  if (in.batch > 0)
    throw Failure{dimension_mismatch, "the resident factor is a batch: download it and solve each problem separately"};
}

// pcg_solve (solver.cpp:95-175) with every reduction, vector update and
// preconditioner sweep in the reference's order: x, the iteration count and
// both residuals are bit-identical to the reference's. The reductions are
// serial chains (O(n) latency each), so this is the default only where that
// is cheap (parac_gpu_pcg, mode 0 with n <= the exact threshold).
void pcg_exact(const SolveInputs& in, double tol, int max_iters, parac_gpu_solve_report& rep) {
  SolveState& s = *in.state;
  const int n = in.n;
  cudaStream_t st = in.stream;
  Solver sv(in);
  const int vb = std::max(1, std::min(kRedBlocks * 2, (n + 255) / 256));
  // rhs = b - mean(b) (b was uploaded into lp); r = rhs; x = 0
  const double mean = sv.chain(kTermSum, s.lp) / static_cast<double>(n);
  center_exact_kernel<<<vb, 256, 0, st>>>(n, s.lp, mean, s.rhs, s.r, s.x);
  note_launches(1);
  const double b_norm = std::sqrt(sv.chain(kTermDot, s.rhs, s.rhs));
  if (b_norm == 0.0) {
    rep.converged = 1;
    return;
  }
  sv.precond(s.r, s.z, kSlotC, true);
  copy_kernel<<<vb, 256, 0, st>>>(n, s.z, s.p);
  copy_kernel<<<vb, 256, 0, st>>>(n, s.x, s.best);
  note_launches(2);
  double rz = sv.chain(kTermDot, s.r, s.z);
  double best_norm = b_norm;  // norm2(r) with r = rhs: the same chain, the same bits
  double rn = b_norm;         // norm2(r) of the current r (loop test, :130)
  int iters = 0;
  while (iters < max_iters) {
    if (rn <= tol * b_norm) break;
    ++iters;
    sv.spmv(s.p, s.lp, kSlotA);
    const double p_lp = sv.chain(kTermDot, s.p, s.lp);
    if (!(p_lp > 0.0)) break;
    const double alpha = rz / p_lp;
    update_xr_exact_kernel<<<vb, 256, 0, st>>>(n, alpha, s.x, s.r, s.p, s.lp);
    note_launches(1);
    // z does not depend on ||r||: the sweep first, then both chains at once
    sv.precond(s.r, s.z, kSlotC, true);
    double two[2];
    sv.chains(Chain{kTermDot, s.r, s.r}, Chain{kTermDot, s.r, s.z}, 2, two);
    rn = std::sqrt(two[0]);
    if (rn < best_norm) {
      best_norm = rn;
      copy_kernel<<<vb, 256, 0, st>>>(n, s.x, s.best);
      note_launches(1);
    }
    const double beta = two[1] / rz;
    rz = two[1];
    update_p_exact_kernel<<<vb, 256, 0, st>>>(n, beta, s.z, s.p);
    note_launches(1);
  }
  double rec = rn;
  if (rec > best_norm) {
    copy_kernel<<<vb, 256, 0, st>>>(n, s.best, s.x);
    note_launches(1);
    rec = best_norm;
  }
  rep.recurrence_residual = rec / b_norm;
  const double xmean = sv.chain(kTermSum, s.x) / static_cast<double>(n);
  center_exact_kernel<<<vb, 256, 0, st>>>(n, s.x, xmean, s.x, nullptr, nullptr);
  note_launches(1);
  sv.spmv(s.x, s.lp, kSlotA);
  rep.iterations = iters;
  rep.relative_residual = std::sqrt(sv.chain(kTermDiff, s.rhs, s.lp)) / b_norm;
  rep.converged = rep.relative_residual <= tol;
}

// Fast PCG (the default above the exact threshold): pcg_solve's control flow
// with fixed-order tree reductions and the fast sweeps. The loop runs on the
// device as a CUDA graph -- a while node whose body is one iteration
// (SpMV, x/r update, the loop test and best-iterate bookkeeping in a one-thread
// control kernel, preconditioner sweeps, p update) -- captured once per factor
// and replayed per solve. PARAC_PCG_GRAPH=0 drives the same kernels from the
// host (one control read per iteration) for comparison.
void pcg_fast(const SolveInputs& in, double tol, int max_iters, parac_gpu_solve_report& rep) {
  SolveState& s = *in.state;
  const int n = in.n;
  cudaStream_t st = in.stream;
  Solver sv(in);
  sv.center(s.lp, s.rhs, s.r, s.x);  // rhs = b - mean, r = rhs, x = 0
  const double b_norm = std::sqrt(sv.read_partials(kSlotB));
  if (b_norm == 0.0) {
    rep.converged = 1;
    return;
  }
  sv.precond(s.r, s.z, kSlotC, false);  // slot C = r0.z0
  copy_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, s.z, s.p);
  copy_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, s.x, s.best);
  note_launches(2);
  double rn = b_norm, best_norm = b_norm;  // norm2(r) with r = rhs
  int iters = 0;
  if (max_iters > 0 && rn > tol * b_norm) {
    const double sc[3] = {b_norm, b_norm, tol * b_norm};  // kRn, kBest, kTolB
    const int ctl[2] = {0, max_iters};
    check(cudaMemcpyAsync(s.scalars + kRn, sc, sizeof(sc), cudaMemcpyHostToDevice, st), "h2d");
    check(cudaMemcpyAsync(s.counters + kCtl, ctl, sizeof(ctl), cudaMemcpyHostToDevice, st), "h2d");
    int* dctl = s.counters + kCtl;
    auto body = [&](cudaGraphConditionalHandle cond, int set_cond) {
      sv.spmv(s.p, s.lp, kSlotA);
      update_xr_g_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, sv.part(kSlotA), sv.part(kSlotC), s.scalars, s.x,
                                                             s.r, s.p, s.lp, sv.part(kSlotB));
      pcg_control_kernel<<<1, 1, 0, st>>>(sv.part(kSlotB), s.scalars, dctl, cond, set_cond);
      copy_if_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, dctl + kCtlCopy, s.x, s.best);
      note_launches(3);
      sv.precond(s.r, s.z, kSlotC, false);
      update_p_g_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, sv.part(kSlotC), s.scalars, s.z, s.p);
      note_launches(1);
    };
    static const bool use_graph = [] {
      const char* e = std::getenv("PARAC_PCG_GRAPH");
      return !(e && std::atoi(e) == 0) && !std::getenv("PARAC_SWEEP_PROFILE");
    }();
    if (use_graph) {
      if (!s.pcg_exec) {
        cudaGraph_t g = nullptr;
        check(cudaGraphCreate(&g, 0), "graph create");
        s.pcg_graph = g;
        cudaGraphConditionalHandle cond;
        check(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault), "conditional handle");
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = cond;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        check(cudaGraphAddNode(&node, g, nullptr, 0, &cp), "while node");
        cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
        const long long l0 = parac_gpu_launch_count();
        check(cudaStreamBeginCaptureToGraph(st, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal),
              "capture");
        body(cond, 1);
        cudaGraph_t captured = nullptr;
        check(cudaStreamEndCapture(st, &captured), "end capture");
        s.pcg_body_launches = parac_gpu_launch_count() - l0;
        note_launches(-s.pcg_body_launches);  // counted per executed iteration below
        check(cudaGraphInstantiate(&s.pcg_exec, g, 0), "graph instantiate");
      }
      check(cudaGraphLaunch(s.pcg_exec, st), "graph launch");
    } else {
      int cont = 1;
      while (cont) {
        body(0, 0);
        check(cudaMemcpyAsync(&cont, dctl + kCtlCopy + 1, sizeof(int), cudaMemcpyDeviceToHost, st), "d2h");
        check(cudaStreamSynchronize(st), "sync");
      }
    }
    double back[2];
    check(cudaMemcpyAsync(back, s.scalars + kRn, sizeof(back), cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaMemcpyAsync(&iters, dctl + kCtlIters, sizeof(int), cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaStreamSynchronize(st), "pcg loop");
    rn = back[0];
    best_norm = back[1];
    if (use_graph) note_launches(s.pcg_body_launches * iters);
  }
  double rec = rn;  // norm2(r) of the final r (:156)
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

// parac_gpu_pcg's mode 0 runs the exact PCG up to this size (PARAC_EXACT_PCG_N)
int exact_pcg_max_n() {
  static const int v = [] {
    const char* e = std::getenv("PARAC_EXACT_PCG_N");
    return e ? std::atoi(e) : 16384;
  }();
  return v;
}

}  // namespace

void solve_release(SolveState& s) {
  drop_pcg_graph(s);
  dfree(s.wdeg); dfree(s.inv); dfree(s.gt_ptr); dfree(s.gt_col); dfree(s.gt_val);
  dfree(s.level); dfree(s.order); dfree(s.lvl_off); dfree(s.flags);
  dfree(s.x); dfree(s.r); dfree(s.p); dfree(s.lp); dfree(s.z); dfree(s.best);
  dfree(s.yf); dfree(s.yd); dfree(s.zb); dfree(s.rhs);
  dfree(s.partials); dfree(s.scalars); dfree(s.counters); dfree(s.tiles); dfree(s.tmp_int);
  dfree(s.hsplit); dfree(s.tail_s); dfree(s.tail_cnt);
  dfree(s.lf_ptr); dfree(s.lb_ptr); dfree(s.lf_idx); dfree(s.lb_idx); dfree(s.lf_val); dfree(s.lb_val);
  dfree(s.lvl_target); dfree(s.ltime);
  dfree(s.lpos); dfree(s.rlab); dfree(s.v2l); dfree(s.dinv_l); dfree(s.rhs_l); dfree(s.hrec_f); dfree(s.hrec_b);
  dfree(s.t3_fep); dfree(s.t3_fidx); dfree(s.t3_fval);
  dfree(s.tw); dfree(s.twt); dfree(s.tw_offl); dfree(s.tw_offu);
  s = SolveState{};
}
void solve_invalidate(SolveState& s) {
  s.graph_ready = false;
  s.components = -1;
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
  NvtxRange nvtx_range("parac_gpu_laplacian_apply");
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
  NvtxRange nvtx_range("parac_gpu_apply_preconditioner");
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
    if (in.state->ltime) {  // diagnostics: [H, depth, tail rows, wide levels] then 16 x (depth+2) stamps
      const SolveState& ss = *in.state;
      std::vector<unsigned long long> t(16 * (static_cast<std::size_t>(ss.depth) + 2));
      check(cudaMemcpy(t.data(), ss.ltime, t.size() * 8, cudaMemcpyDeviceToHost), "d2h");
      if (FILE* f = std::fopen(std::getenv("PARAC_SWEEP_PROFILE"), "wb")) {
        const int hdr[4] = {ss.t3_L0, ss.depth, ss.t3_nt, std::min(ss.wide_L, ss.t3_L0)};
        std::fwrite(hdr, 4, 4, f);
        std::fwrite(t.data(), 8, t.size(), f);
        std::fclose(f);
      }
    }
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
  NvtxRange nvtx_range("parac_gpu_schedule_levels");
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
  NvtxRange nvtx_range("parac_gpu_pcg");
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
    parac_gpu_solve_report rep{};
    struct Events {  // destroyed on every path out (a failed check throws)
      cudaEvent_t e[2] = {nullptr, nullptr};
      ~Events() {
        for (cudaEvent_t x : e)
          if (x) cudaEventDestroy(x);
      }
    } ev;
    check(cudaEventCreate(&ev.e[0]), "event");
    check(cudaEventCreate(&ev.e[1]), "event");
    cudaEvent_t e0 = ev.e[0], e1 = ev.e[1];
    check(cudaEventRecord(e0, st), "event");

    upload(s.lp, b, n, st);
    const bool exact = s.mode == kModeExact || (s.mode == kModeDefault && n <= exact_pcg_max_n());
    rep.exact = exact ? 1 : 0;
    if (exact) pcg_exact(in, tol, max_iters, rep);
    else pcg_fast(in, tol, max_iters, rep);
    check(cudaEventRecord(e1, st), "event");
    check(cudaGetLastError(), "pcg");
    download(x, s.x, n, st);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    rep.solve_ms = ms;
    rep.wall_ms = wall.ms();
    if (report) *report = rep;
  });
}

}  // extern "C"
