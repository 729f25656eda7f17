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
// Capacity of a small warp's column scratch. The routing threshold itself is
// FactorDev::small_cap (<= kSmallCap), chosen per problem: 64 on sparse
// meshes, where a 65-128 entry column took ~20 us on one warp (two 4-item
// sorts on 32 lanes) vs ~10 us on a CTA and such columns are ~40% of the
// 128^3 critical path (tools/profile_factor.py, by_raw); 128 on denser
// graphs (27-point), where they are common enough in the wide phase that the
// big-CTA pool would become the throughput limit (96 measured best there:
// 27-point 96^3 K3 31.3 ms vs 32.9 at 128 and 35.3 at 64). A capacity of 96
// rather than 128 keeps the small path's sample/decrement batches at 3 per
// lane (fewer registers: 128^3 K3 19.5 vs 20.2 ms with the same routing).
constexpr int kSmallCap = 96;
// vertices of higher degree get a whole CTA in the forward-graph build (K1)
constexpr int kHeavyDeg = 64;
// wide-column slab (cooperative hub path, eliminate.cu): 7 arrays of 8 B per
// entry -- raw keys/weights (tile-sorted, then the merged column), sorted raw
// keys/weights (then the weight-sorted tiles), weight-ordered column, suffix
constexpr int kSlabEntryBytes = 56;
constexpr int kBigCap = 1024;

// Cooperative wide columns (raw size > kBigCap, R-MAT hubs). The big CTA that
// claims such a column (the owner) runs its elimination as a sequence of
// phases, each cut into 256-entry chunks and posted as a job; big CTAs that
// are waiting for a queue slot take chunks (helpers). The owner takes chunks
// too, so a column finishes with or without helpers.
struct HubDesc {                // one phase of one column (read by every chunk)
  int k, R, m, nt, mt, fdeg, lvk, cs, phase, cap, trace, pipe;  // pipe: sampling follows the suffix chain
  long long fb, slab, start;
  double lkk;
  unsigned dirrow[kDirChunks];
};
struct HubJob {  // one per CTA of the elimination grid
  // seq << 48 | nchunks << 24 | chunks claimed: claiming a chunk is one
  // atomicAdd, and the returned word says which phase the chunk belongs to
  alignas(256) unsigned long long next;
  alignas(256) unsigned long long done;  // seq << 32 | chunks completed
  alignas(256) HubDesc desc[2];          // by seq parity
  alignas(256) int emitted;              // fills emitted by the sampling phase
  alignas(256) int progress;             // suffix sums C[progress, m) are written (pipelined sampling)
};
// Optional per-column trace of the hub path (record_times; tools/profile_factor.py):
// [0] k [1] R [2] m [3] owner start [4] owner end (globaltimer ns), then per
// step p = 1..9 (7 phases, 8 = lkk chain, 9 = suffix chain) at 8 + 4 (p - 1):
// posted, first chunk started, last chunk ended, owner chunks << 32 | helper chunks;
// at 48 + p (p = 1..7): the sum of the phase's chunk durations (ns)
constexpr int kHubTraceWords = 64;
// Ctrl::status when a column wider than kBigCap met the kernel instance
// without the hub path: the host re-runs with it (never returned to callers)
constexpr int kStatusNeedHubs = 90;
constexpr int kHubTraceCap = 1 << 16;

// Control block. The counters every elimination touches (queue heads and
// tails, the column arena bump, the eliminated count, the status word the
// waiters poll) each get their own 256-byte line: sharing one line serialised
// the wide phase's ~800 atomics/us at a single L2 slice (measured: a relaxed
// load of q_head/q_tail alongside the decrements cost ~3 us).
struct Ctrl {
  alignas(256) int status;  // 0 or Errc
  alignas(256) int q_head;  // main (small-column) queue: next slot to claim
  alignas(256) int q_tail;  //                            next slot to publish
  alignas(256) int b_head;  // big-column queue
  alignas(256) int b_tail;
  alignas(256) int eliminated;               // vertices done (flushed per warp before it waits)
  alignas(256) unsigned long long arena_bump;  // G column arena (entries)
  alignas(256) int max_raw;                  // largest gathered column
  int large_cols;                            // columns that used the global-memory slab
  unsigned long long ovf_bump;               // fill overflow pool (entries)
  unsigned long long large_bump;             // large-column slab pool (entries)
  long long total_fills;
  long long err_info;
  alignas(256) int sm_slot[256];             // CTAs started per SM (role assignment)
  alignas(256) int hub_hint;                 // job index + 1 of the latest posted hub phase (0: none)
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
  // large-column slab pool: kSlabEntryBytes per entry
  char* large_pool;
  long long large_cap;
  HubJob* hub_jobs;  // [grid] cooperative wide-column jobs, one per CTA
  unsigned long long* hub_trace;  // optional [kHubTraceCap * kHubTraceWords]
  unsigned long long hub_linger_ns;  // a helper waits this long for a job's next phase
  unsigned hub_wait_ns;              // longest sleep of a waiting big CTA between looks at the hub hint
  int hubs;          // launch the kernel with the cooperative hub path (hub graphs; see launch_eliminate)
  int hub_pipe;      // hub columns: sampling starts while the suffix chain runs (1; PARAC_HUB_PIPE=0 off)
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
  int big_layout;        // 0: every 4th SM runs big CTAs only; 1: one big CTA per SM
  int small_cap;         // columns with more raw entries go to the big-CTA queue (<= kSmallCap)
  int discard_fills;     // drop a column's fill-slot L2 lines once it has gathered them
  unsigned long long* vtimes;  // optional [8n] phase timestamps per position
  unsigned long long* vsub;    // optional [8n] sub-phase timestamps per position
  // optional TestHooks::on_phase analogue: dp snapshots [3n] at the phase
  // boundaries of position trace_k's elimination (trace_k < 0: off)
  int trace_k;
  long long* trace_dp;
  int* trace_taken;
  // streamed assembly (stream_assemble.cu): eliminated columns per block of
  // kStreamBlock positions, one relaxed add per column after its release
  // fence; nullptr when the assembly runs after the elimination
  int* blk_done;
};

// Streamed CSC assembly beside K3 (stream_assemble.cu).
constexpr int kStreamShift = 11;
constexpr int kStreamBlock = 1 << kStreamShift;
struct StreamDev {
  int n, nb;                        // positions, blocks
  int start_after;                  // begin once K3 has eliminated this many positions
  const int* blk_done;              // [nb] eliminated columns per block (K3)
  const int* col_len;
  const long long* col_start;
  const int* arena_rows;
  const double* arena_vals;
  long long* col_ptr;               // the resident CSC factor (as launch_assemble writes it)
  int* rows;
  double* vals;
  unsigned long long* blk_incl;     // [nb] block total | bit 62, then inclusive entry offset | bit 63
  int* next_blk;                    // block claim counter
  unsigned long long* host_blk;     // [nb] mapped pinned: inclusive entry end | bit 63 once released
  Ctrl* ctrl;                       // status (K3 aborted), eliminated
  // batch (disjoint union): blocks never straddle problems -- block b is
  // positions [blk_k0[b], blk_k0[b+1]) (nullptr: b * kStreamBlock); rows are
  // made local to their problem (pos_pid / pid_base)
  const int* blk_k0;
  const int* pos_pid;
  const long long* pid_base;
  // batch regions (optional): member p's entries at region[p] + its local
  // offsets (capacity reg_cap[p]; beyond it *overflow = 1 and the block is not
  // copied), its local col_ptr at lcol[base_p + p ...]; offsets by look-back
  // within the member (blk_first[b] = its first block); blocks claimed in the
  // order claim[] (members interleaved)
  const int* claim;
  const int* blk_first;
  const long long* region;
  const long long* reg_cap;
  long long* lcol;
  int* overflow;
};
cudaError_t launch_stream_assemble(const StreamDev& s, int ctas, cudaStream_t st);
cudaError_t launch_sum_samples(const FactorDev& d, cudaStream_t s);

// Launchers (stream-ordered). All return cudaError_t of the launch.
cudaError_t launch_pos_graph(const FactorDev& d, long long* tile_scratch, cudaStream_t s);
cudaError_t launch_initial_ready(const FactorDev& d, long long* tile_scratch, cudaStream_t s);
int initial_ready_scratch(int n);  // long longs of tile_scratch launch_initial_ready needs
cudaError_t launch_eliminate(const FactorDev& d, int grid_ctas, int reserve, cudaStream_t s, int* grid_used);
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
