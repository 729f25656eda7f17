// Device PCG state (solve path): SpMV, level-synchronous triangular sweeps
// (fast mode: wide levels / cluster head / dense-inverse tail; exact mode: cluster),
// fused vector ops. See solve_kernels.cu.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

struct parac_gpu_ctx;

namespace parac_gpu {

struct SolveState {
  bool graph_ready = false;   // wdeg computed for the staged graph
  int components = -1;        // connected components of the staged graph (-1: not yet counted)
  bool factor_ready = false;  // G^T (CSR), inverse perm, level order built
  int n = 0;
  double* wdeg = nullptr;
  int* inv = nullptr;
  // G in row form (CSR over positions): entries (k, G(r,k)), k ascending
  long long* gt_ptr = nullptr;
  int* gt_col = nullptr;
  double* gt_val = nullptr;
  int* level = nullptr;       // forward ASAP level per position
  int* order = nullptr;       // positions sorted by level
  long long* lvl_off = nullptr;  // level offsets into order
  int* flags = nullptr;       // completion stamps per position (level pass)
  // fast-mode one-CTA tail (levels > t3_L0): tail rows' right-hand side after
  // the head's contributions, scratch counts and forward T-part offsets
  long long* hsplit = nullptr;
  double* tail_s = nullptr;
  int* tail_cnt = nullptr;
  // G's rows (forward) / columns (backward) copied in level order
  long long *lf_ptr = nullptr, *lb_ptr = nullptr;
  int *lf_idx = nullptr, *lb_idx = nullptr;
  double *lf_val = nullptr, *lb_val = nullptr;
  long long* lvl_target = nullptr;
  unsigned long long* ltime = nullptr;  // PARAC_SWEEP_PROFILE: per-level timestamps
  // v3 fast sweeps (level-order index space): maps, head chunk tables, tail arrays
  int *lpos = nullptr, *rlab = nullptr, *v2l = nullptr;
  double *dinv_l = nullptr, *rhs_l = nullptr;
  int4 *hrec_f = nullptr, *hrec_b = nullptr;
  int head_csize = 0, head_W = 0;
  int wide_L = 0;                             // the wide first levels (one launch per level)
  std::vector<long long> lvl_off_h;           // host copy of the level offsets of levels 0..wide_L+1
  std::vector<int> wide_kf, wide_kb;          // lanes per row of each wide level (forward rows / backward columns)
  // dense-inverse tail (levels > t3_L0, rows t3_base.. in level order, T = t3_nt)
  int t3_L0 = 0, t3_nt = 0, t3_base = 0, t3_nlev = 0;
  int *t3_fep = nullptr, *t3_fidx = nullptr;  // tail rows' entries inside the tail (tail-relative)
  double* t3_fval = nullptr;
  double *tw = nullptr, *twt = nullptr;       // W = G_TT^-1 (lower packed) and W^T (rows = W's columns)
  long long *tw_offl = nullptr, *tw_offu = nullptr;
  int tw_T = 0, tw_Tp = 0;
  std::size_t cap_tw = 0, cap_twt = 0;
  std::size_t cap_v3 = 0, cap_hrec = 0, cap_t3 = 0, cap_t3e = 0;
  std::size_t cap_ltime = 0;
  std::size_t cap_lz = 0, cap_levels = 0;
  // fast PCG loop as a CUDA graph (a while node over one iteration), built on
  // the first solve of a factor and replayed: no host round trip per iteration
  cudaGraphExec_t pcg_exec = nullptr;
  cudaGraph_t pcg_graph = nullptr;
  long long pcg_body_launches = 0;
  int mode = 0;  // 0 default (pcg fast, apply exact), 1 exact, 2 fast
  int depth = 0;
  int epoch = 0;
  // vectors
  double *x = nullptr, *r = nullptr, *p = nullptr, *lp = nullptr, *z = nullptr, *best = nullptr;
  double *yf = nullptr, *yd = nullptr, *zb = nullptr, *rhs = nullptr;
  double* partials = nullptr;  // per-block partial sums
  double* scalars = nullptr;   // device scalars
  int* counters = nullptr;     // claim counters
  long long* tiles = nullptr;
  int* tmp_int = nullptr;
  std::size_t cap_n = 0, cap_z = 0;
  int blocks = 0;
};

enum : int { kModeDefault = 0, kModeExact = 1, kModeFast = 2 };

struct SolveInputs {
  int n;
  const long long* ptr;
  const int* adj;
  const double* w;
  int f_n;
  long long f_nnz;
  const long long* col_ptr;
  const int* rows;
  const double* vals;
  const double* diag;
  const int* perm;
  const int* level;  // ASAP levels from K3 (nullptr: compute them)
  int batch;         // >0: the resident factor is a batch (per-problem rows); no solve
  cudaStream_t stream;
  int device;
  SolveState* state;
};

void solve_release(SolveState& s);
void solve_invalidate(SolveState& s);
void solve_invalidate_factor(SolveState& s);
SolveInputs solve_inputs(parac_gpu_ctx* ctx);
void ctx_activate(parac_gpu_ctx* ctx);

}  // namespace parac_gpu
