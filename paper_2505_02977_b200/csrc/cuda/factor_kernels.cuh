// Device state and launch interface of the factorization path.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace parac_gpu {

// Fill entries are 16 B {row, source, weight}: one v4 store / load.
// Fill storage per vertex (position) lo:
//   slots [0, C0)                     -> pool0[lo*C0 + s]      (preallocated)
//   chunk c>=1: slots [C0(2^c-1), C0(2^(c+1)-1)) -> ovf[(dir[lo][c-1]-1)*C0 ...]
//   chunks are bump-allocated on first touch by the writer of their first slot.
constexpr int kDirChunks = 16;

// Two warp tiers in the persistent elimination kernel: "small" warps hold
// columns of up to kSmallCap raw entries in shared memory, one "big" warp per
// CTA holds up to kBigCap (wider columns use a global-memory slab). A vertex is
// routed to the matching ready queue when it becomes ready.
constexpr int kSmallCap = 128;
// vertices of higher degree get a whole CTA in the forward-graph build (K1)
constexpr int kHeavyDeg = 64;
// wide-column slab: A (u64), B (f64), C (f64), A2, B2 per entry
constexpr int kSlabEntryBytes = 40;
constexpr int kBigCap = 1024;

struct Ctrl {
  int status;            // 0 or Errc
  int q_head;            // main (small-column) queue: next slot to claim
  int q_tail;            //                            next slot to publish
  int b_head;            // big-column queue
  int b_tail;
  int eliminated;        // vertices done (flushed per warp before it waits)
  int max_raw;           // largest gathered column
  int large_cols;        // columns that used the global-memory slab
  unsigned long long ovf_bump;    // fill overflow pool (entries)
  unsigned long long arena_bump;  // G column arena (entries)
  unsigned long long large_bump;  // large-column slab pool (entries)
  long long total_fills;
  long long err_info;
  int pad0;
  int pad1;
};

struct FactorDev {
  int n;
  // label-space input (LaplacianGraph CSR) + ordering
  const long long* ptr;
  const int* adj;
  const double* w;
  const int* perm;
  // position-space forward graph (PosGraph, factor_common.hpp:23-29)
  int* inv;
  long long* fwd_ptr;
  int* fwd_to;
  double* fwd_w;
  int* fdeg;
  int* heavy_list;     // labels with degree > kHeavyDeg (K1), count in *heavy_count
  int* heavy_count;
  int* heavy_key;      // K1 hub sort scratch, same offsets as fwd_to / fwd_w
  double* heavy_val;
  // dependency counters + ready queues
  // per-position counters, one 64-bit word each: low 32 bits = dp (pending
  // earlier neighbours + pending fill endpoints), high 32 bits = fills
  // received. One word means the decrement that makes a vertex ready also
  // returns its final fill count -- no extra round trip, no extra fence.
  unsigned long long* cnt;
  int* queue;   // main queue [n]
  int* bqueue;  // big-column queue [n]
  int keep_pos; // keep-one preference: 0 widest column, 1 lowest position
  // fills
  int4* pool0;
  unsigned* dir;
  int4* ovf;
  long long ovf_cap;
  int c0;
  // G columns (arena, then assembled into CSC)
  long long* col_start;
  int* col_len;
  double* diag;
  int* arena_rows;
  double* arena_vals;
  long long arena_cap;
  int* samples;
  int* level;  // optional: ASAP level per position (schedule_levels), 1-based
  // large-column slab pool: 24 B per entry
  char* large_pool;
  long long large_cap;
  // control
  Ctrl* ctrl;
  unsigned long long sample_seed;
  // batch (disjoint union of problems): problem of each position, its first
  // position and its derived sample seed; pos_pid == nullptr for one problem
  const int* pos_pid;
  const long long* pid_base;
  const unsigned long long* pid_seed;
  unsigned long long watchdog_ns;
  int verify;
  int delay_ns;
  unsigned sleep_ns[3];  // claim() backoff by distance to the publishing front (16-256, 256-1024, >1024 slots)
  int keep_limit;        // max consecutive keep-one hand-offs before a warp/CTA returns to the queue
  unsigned long long* vtimes;  // optional [8n] phase timestamps per position
  unsigned long long* vsub;    // optional [8n] sub-phase timestamps per position
};

// Launchers (stream-ordered). All return cudaError_t of the launch.
cudaError_t launch_pos_graph(const FactorDev& d, long long* tile_scratch, cudaStream_t s);
cudaError_t launch_initial_ready(const FactorDev& d, long long* tile_scratch, cudaStream_t s);
int initial_ready_scratch(int n);  // long longs of tile_scratch launch_initial_ready needs
cudaError_t launch_eliminate(const FactorDev& d, int grid_ctas, cudaStream_t s, int* grid_used);
cudaError_t launch_assemble(const FactorDev& d, long long* col_ptr, int* rows, double* vals,
                            long long* tile_scratch, cudaStream_t s);
cudaError_t launch_scan(const int* in, long long n, long long* out, long long* tile_scratch,
                        cudaStream_t s);
long long scan_tiles(long long n);
int eliminate_occupancy_grid(int device);
// batch (disjoint union): add label / edge offsets to the staged union, and
// rebase each problem's factor rows to its own position space
cudaError_t launch_batch_offsets(int count, long long N, long long NNZ, const long long* base,
                                 const long long* ebase, long long* ptr, int* adj, int* perm, int* pos_pid,
                                 cudaStream_t s);
// fills_received per position (high words of cnt) into out[n]
cudaError_t launch_extract_fills(int n, const unsigned long long* cnt, int* out, cudaStream_t s);
cudaError_t launch_batch_local_rows(int n, const long long* col_ptr, const int* pos_pid, const long long* base,
                                    int* rows, cudaStream_t s);
// ordering_nnz_sort on the device (ordering.cu): perm from the CSR row pointer
void nnz_sort_device(int n, const long long* d_ptr, std::uint64_t tie_seed, int* d_perm, cudaStream_t st, int sms);
void max_degree_device(int n, const long long* d_ptr, long long* d_out, cudaStream_t st, int sms);

}  // namespace parac_gpu
