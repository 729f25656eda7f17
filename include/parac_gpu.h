/*
 * parac_gpu.h — C ABI of the B200-native (sm_100a) randomized approximate
 * Cholesky (rchol / ParAC, arXiv 2505.02977) factorization of graph
 * Laplacians and the PCG solve that consumes it.
 *
 * This is the drop-in boundary for the reference library `parac`
 * (/root/reference/proj). Each entry point names the reference interface it
 * replaces (file:line, paths relative to proj/). Conventions:
 *   - plain pointers and sizes only, no C++ or torch types;
 *   - every fallible call returns an int status: 0 = ok, otherwise the
 *     reference's `parac::Errc` value (include/parac/error.hpp:9-27), so a C++
 *     shim can rethrow `parac::Error(Errc(code), parac_gpu_last_error())`;
 *   - inputs are never owned; outputs go to caller buffers (or are freed by
 *     the matching *_free call);
 *   - there is NO CPU fallback: without a CUDA device every device entry point
 *     fails with PARAC_INTERNAL_ERROR and a message saying so.
 * See INTEGRATION.md for the C++ shim (parac::factor_gpu / pcg_solve_gpu).
 */
#ifndef PARAC_GPU_H
#define PARAC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: identical numbering to parac::Errc (error.hpp:9-27) ---- */
enum {
  PARAC_OK = 0,
  PARAC_ASYMMETRIC_INPUT = 1,
  PARAC_POSITIVE_OFF_DIAGONAL = 2,
  PARAC_ROW_SUM_VIOLATION = 3,
  PARAC_TOO_LARGE_FOR_DENSE = 4,
  PARAC_PARSE_ERROR = 5,
  PARAC_UNSUPPORTED_FIELD = 6,
  PARAC_BUDGET_EXCEEDED = 7,
  PARAC_NOT_A_PERMUTATION = 8,
  PARAC_DENSE_BLOWUP = 9,
  PARAC_ARENA_EXHAUSTED = 10,
  PARAC_QUEUE_STALL = 11,
  PARAC_WORKSPACE_FULL = 12,
  PARAC_DIMENSION_MISMATCH = 13,
  PARAC_NOT_CONNECTED = 14,
  PARAC_TOO_MANY_NEIGHBORS = 15,
  PARAC_IO_ERROR = 16,
  PARAC_INTERNAL_ERROR = 17
};

/* errc_name (src/error.cpp:5-27): "ArenaExhausted", ... */
const char* parac_errc_name(int code);
/* Message of the last failing call on this host thread. */
const char* parac_gpu_last_error(void);

/* ---- graphs: LaplacianGraph (include/parac/graph.hpp:25-60) as CSR ---------
 * Label space, neighbours ascending within a row, weights > 0, both halves
 * stored (nnz = ptr[n] = 2E). wdeg (the derived diagonal) is optional on
 * input; the library recomputes it in the reference's order when needed. */
typedef struct {
  int32_t n;
  const int64_t* ptr; /* n+1 */
  const int32_t* adj; /* ptr[n] */
  const double* w;    /* ptr[n] */
} parac_csr;

/* Library-owned CSR produced by the host builders below. */
typedef struct {
  int32_t n;
  int64_t nnz; /* = ptr[n] */
  int64_t* ptr;
  int32_t* adj;
  double* w;
  double* wdeg;
} parac_graph;
void parac_graph_free(parac_graph* g);

/* LaplacianGraph::from_edges (graph.hpp:33, src/graph.cpp:21-83): unique
 * undirected edges (a_i != b_i), w_i > 0; rejects self-loops, non-positive
 * weights, out-of-range endpoints and duplicates with PARAC_INTERNAL_ERROR. */
int parac_graph_from_edges(int32_t n, int64_t m, const int32_t* a, const int32_t* b,
                           const double* w, parac_graph* out);

/* gen_poisson3d (generators.hpp:26, src/generators.cpp:14-65).
 * variant: 0 uniform, 1 anisotropic (z-edges epsilon), 2 contrast. */
int parac_gen_poisson3d(int32_t n, int variant, double epsilon, double contrast_ratio,
                        uint64_t seed, parac_graph* out);
/* 2D 5-point n x n grid, unit weights, id = x + n*y (BASELINE config 1). */
int parac_gen_poisson2d(int32_t n, parac_graph* out);
/* 3D 27-point (Chebyshev distance 1) n^3 grid, w(a,b) = 0.5 + 1.5 *
 * unit_uniform(derive_seed(seed, kSaltCells), a, b) for a < b (config 3). */
int parac_gen_poisson27(int32_t n, uint64_t seed, parac_graph* out);
/* R-MAT (Graph500 a,b,c = .57,.19,.19), 2^scale vertices, edge_factor *
 * 2^scale samples, self-loops dropped, deduplicated, w in U[0.5,2) keyed by
 * (u,v) (config 4). */
int parac_gen_rmat(int32_t scale, int32_t edge_factor, uint64_t seed, parac_graph* out);
/* gen_random_connected / gen_random_components (src/generators.cpp:110-175),
 * same SplitMix64 streams, so the graphs equal the reference's. */
int parac_gen_random_connected(int32_t n, int64_t extra_edges, uint64_t seed,
                               int unit_weights, parac_graph* out);
int parac_gen_random_components(int32_t n, int32_t components, int64_t extra_edges,
                                uint64_t seed, parac_graph* out);

/* ---- orderings: Ordering::perm (include/parac/ordering.hpp:13-24) ---------
 * perm[label] = elimination position. */
/* ordering_random (ordering.hpp:28, src/ordering.cpp:38-47) */
int parac_ordering_random(int32_t n, uint64_t seed, int32_t* perm);
/* ordering_nnz_sort (ordering.hpp:32, src/ordering.cpp:49-70) */
int parac_ordering_nnz_sort(const parac_csr* g, uint64_t seed, int32_t* perm);
/* Ordering::from_positions validation (src/ordering.cpp:22-36):
 * PARAC_NOT_A_PERMUTATION unless perm is a bijection on [0,n). */
int parac_ordering_check(int32_t n, const int32_t* perm);

/* ---- Matrix Market text I/O (include/parac/matrix_market.hpp) -------------
 * Byte-identical files to the reference writers (values as %.17g, exact
 * binary64 round trip); readers accept what the reference readers accept and
 * fail with the same Errc (PARAC_IO_ERROR, PARAC_PARSE_ERROR "<path>:<line>:
 * what", PARAC_UNSUPPORTED_FIELD, validate_laplacian's codes). Formatting and
 * parsing run on all host threads. */
/* read_laplacian (src/matrix_market.cpp:129-135) = read_matrix_market (:65-127)
 * + validate_laplacian (src/graph.cpp:99-186) -> library-owned graph. */
int parac_read_laplacian(const char* path, parac_graph* out);
/* write_matrix_market (src/matrix_market.cpp:137-159): symmetric lower
 * triangle, row major, diagonal (weighted degree) first. */
int parac_write_matrix_market(const char* path, const parac_csr* g);
/* write_factor (src/matrix_market.cpp:161-184): <stem>.G.mtx (coordinate
 * real general, strictly lower, 1-based) and <stem>.D.mtx (array real). */
int parac_write_factor(const char* stem, int32_t n, const int64_t* col_ptr, const int32_t* rows,
                       const double* values, const double* diag);
/* Library-owned LdlFactor arrays (include/parac/factor.hpp:18-25). */
typedef struct {
  int32_t n;
  int64_t nnz; /* off-diagonal = col_ptr[n] */
  int64_t* col_ptr;
  int32_t* rows;
  double* values;
  double* diag;
  int32_t* perm;
} parac_factor;
void parac_factor_free(parac_factor* f);
/* read_factor (src/matrix_market.cpp:186-266): columns sorted by (row,
 * value); perm from ordering_from_file(perm_path) or identity when
 * perm_path is NULL or "". */
int parac_read_factor(const char* stem, const char* perm_path, parac_factor* out);
/* write_vector / read_vector (src/matrix_market.cpp:268-304). read_vector
 * returns a malloc'd array (free with parac_free_array). */
int parac_write_vector(const char* path, int64_t n, const double* values);
int parac_read_vector(const char* path, double** values, int64_t* n);
void parac_free_array(void* p);
/* write_permutation / ordering_from_file + Ordering::from_positions
 * (src/ordering.cpp:72-93, :22-36): one position per line. */
int parac_write_permutation(const char* path, int32_t n, const int32_t* perm);
int parac_read_permutation(const char* path, int32_t n, int32_t* perm);

/* ---- device context --------------------------------------------------------
 * Owns the device buffers (reused across calls, grown on demand) and a CUDA
 * stream. Re-entrant per context; use one context per concurrent problem
 * (e.g. one per GPU / per stream for the batch configuration). */
typedef struct parac_gpu_ctx parac_gpu_ctx;
int parac_gpu_create(int32_t device, parac_gpu_ctx** out);
void parac_gpu_destroy(parac_gpu_ctx* ctx);
/* Number of visible CUDA devices (0 on a CPU-only host). */
int parac_gpu_device_count(void);

/* Mirrors ParOptions (include/parac/factor_par.hpp:31-45). */
typedef struct {
  int64_t fill_pool_entries;     /* overflow fill pool (16 B entries); <0: default */
  int64_t column_arena_entries;  /* G column arena; <0: default */
  int32_t first_chunk;           /* preallocated fill slots per vertex; <=0: default */
  double watchdog_seconds;       /* <=0: 60 s (ParOptions::watchdog_seconds) */
  int32_t record_stats;          /* keep merged_degree/samples/fills per position */
  int32_t verify;                /* device-side TestHooks::verify analogue */
  int32_t grid_ctas;             /* persistent-kernel CTAs; <=0: occupancy-sized */
  int32_t delay_ns;              /* >0: random __nanosleep injection (TestHooks::delay) */
  int32_t record_times;          /* ParOptions::record_vertex_times: start/end per position */
  int32_t trace_phases;          /* != 0: TestHooks::on_phase analogue -- snapshot every dependency
                                    counter at the phase boundaries of trace_position's elimination */
  int32_t trace_position;        /* the position traced when trace_phases != 0 */
} parac_gpu_options;
void parac_gpu_default_options(parac_gpu_options* opt);

/* FactorStats (include/parac/factor_seq.hpp:22-30) scalars + timings. */
typedef struct {
  int32_t n;
  int64_t num_edges;        /* E = nnz_lower */
  int64_t nnz_off_diagonal; /* Z; LdlFactor::nnz() = Z + n */
  int64_t total_fills;      /* F */
  int64_t fill_pool_used;   /* overflow pool entries used */
  int64_t arena_used;       /* column arena entries used (= Z) */
  int32_t max_raw;          /* largest gathered column (edges + fills) */
  int32_t large_columns;    /* columns that took the large-column path */
  double setup_ms;          /* device: forward-CSR build + dependency init */
  double eliminate_ms;      /* device: persistent elimination kernel */
  double assemble_ms;       /* device: CSC assembly */
  double device_ms;         /* device total (events around all factor kernels), summed over
                               every attempt when default budgets had to grow and retry */
  double upload_ms;         /* host->device copy (0 for resident inputs) */
  double wall_ms;           /* host wall clock of the call */
  int32_t attempts;         /* device passes run (> 1: library-chosen budgets were grown, or the
                               kernel instance with the hub path was needed) */
} parac_gpu_factor_info;

/* Stage graph + ordering on the device of ctx (host->device copy). */
int parac_gpu_upload(parac_gpu_ctx* ctx, const parac_csr* g, const int32_t* perm);

/* Factor the staged input; the factor stays resident in ctx.
 * Replaces factor_parallel_left/right (include/parac/factor_par.hpp:53-62)
 * and factor_randomized (factor_seq.hpp:34-36): byte-identical LdlFactor
 * (LdlFactor::same_values, src/factor.cpp:10-13) for the same graph,
 * ordering and seed. Errors: PARAC_ARENA_EXHAUSTED (pool/arena budget),
 * PARAC_QUEUE_STALL (device watchdog), PARAC_DIMENSION_MISMATCH. */
int parac_gpu_factor_resident(parac_gpu_ctx* ctx, uint64_t seed, const parac_gpu_options* opt,
                              parac_gpu_factor_info* info);

/* One call: upload + factor (the drop-in for factor_parallel_left). */
int parac_gpu_factor(parac_gpu_ctx* ctx, const parac_csr* g, const int32_t* perm, uint64_t seed,
                     const parac_gpu_options* opt, parac_gpu_factor_info* info);

/* The factorization split in two, so that the host can work while the device
 * factors: _begin launches it (returns at once); _end waits for it and copies
 * the factor out WHILE the elimination runs -- each column is copied as soon
 * as it and every column before it are final (the CSC assembly is streamed
 * beside the elimination). Together they replace factor_parallel_left
 * (include/parac/factor_par.hpp:53-62) returning its LdlFactor
 * (include/parac/factor.hpp:18-25): col_ptr[n+1], rows/values[capacity],
 * diag[n], any of them NULL. The factor stays resident either way. Errors as
 * parac_gpu_factor_resident; PARAC_BUDGET_EXCEEDED when Z > capacity (rows/
 * values incomplete, info->nnz_off_diagonal = Z: size them and call
 * parac_gpu_download). Pinned outputs are filled by DMA, pageable ones
 * through pinned staging. */
int parac_gpu_factor_begin(parac_gpu_ctx* ctx, uint64_t seed, const parac_gpu_options* opt);
int parac_gpu_factor_end(parac_gpu_ctx* ctx, parac_gpu_factor_info* info, int64_t* col_ptr, int32_t* rows,
                         double* values, double* diag, int64_t capacity);
/* upload + factor_begin + factor_end: one call from host input to host factor. */
int parac_gpu_factor_to_host(parac_gpu_ctx* ctx, const parac_csr* g, const int32_t* perm, uint64_t seed,
                             const parac_gpu_options* opt, parac_gpu_factor_info* info, int64_t* col_ptr,
                             int32_t* rows, double* values, double* diag, int64_t capacity);

/* ---- batch (BASELINE config[4]: many independent Laplacians per GPU) ------
 * Stage `count` problems (graph i, ordering perms[i], seed seeds[i]) as one
 * disjoint-union problem so a single persistent elimination factors all of
 * them concurrently; every problem's factor is byte-identical to its
 * stand-alone parac_gpu_factor (same graph, ordering and seed). There is no
 * reference entry point for a batch: the reference loops over
 * factor_randomized / factor_parallel_left, one problem at a time. */
int parac_gpu_upload_batch(parac_gpu_ctx* ctx, int32_t count, const parac_csr* graphs,
                           const int32_t* const* perms, const uint64_t* seeds);
/* upload_batch + factor_resident. */
int parac_gpu_factor_batch(parac_gpu_ctx* ctx, int32_t count, const parac_csr* graphs,
                           const int32_t* const* perms, const uint64_t* seeds, const parac_gpu_options* opt,
                           parac_gpu_factor_info* info);
/* The batch counterpart of parac_gpu_factor_end (after parac_gpu_upload_batch +
 * parac_gpu_factor_begin): every member's LdlFactor arrays, in its own position
 * space, copied out while the union is factored. Arrays of `count` pointers
 * (any array or entry may be NULL); capacities[i] = entries of rows[i] /
 * values[i]. PARAC_BUDGET_EXCEEDED when a member's Z exceeds its capacity
 * (the factor stays resident: parac_gpu_batch_nnz + parac_gpu_download_batch). */
int parac_gpu_factor_batch_end(parac_gpu_ctx* ctx, parac_gpu_factor_info* info, int64_t* const* col_ptrs,
                               int32_t* const* rows, double* const* values, double* const* diags,
                               const int64_t* capacities);
/* upload_batch + factor_begin + factor_batch_end. */
int parac_gpu_factor_batch_to_host(parac_gpu_ctx* ctx, int32_t count, const parac_csr* graphs,
                                   const int32_t* const* perms, const uint64_t* seeds, const parac_gpu_options* opt,
                                   parac_gpu_factor_info* info, int64_t* const* col_ptrs, int32_t* const* rows,
                                   double* const* values, double* const* diags, const int64_t* capacities);
/* Off-diagonal count of problem i's factor (size its rows/values buffers). */
int parac_gpu_batch_nnz(parac_gpu_ctx* ctx, int32_t i, int64_t* nnz_off);
/* Problem i's LdlFactor arrays, in its own position space. */
int parac_gpu_download_batch(parac_gpu_ctx* ctx, int32_t i, int64_t* col_ptr, int32_t* rows,
                             double* values, double* diag);

/* Copy the resident factor to caller buffers (LdlFactor fields,
 * include/parac/factor.hpp:18-25): col_ptr[n+1], rows[Z], values[Z],
 * diag[n]; stats arrays [n] may be NULL (need record_stats). */
int parac_gpu_download(parac_gpu_ctx* ctx, int64_t* col_ptr, int32_t* rows, double* values,
                       double* diag, int32_t* merged_degree, int32_t* samples_emitted,
                       int32_t* fills_received);

/* Per-position elimination phase timestamps (%globaltimer ns) of the last
 * factor run with record_times set: start_end[8*k + i], i = 0 start, 1 gathered
 * and sorted, 2 merged, 3 column written, 4 weight-sorted + suffix, 5 fills
 * emitted, 6 decremented, 7 end (after publishing). Zero = phase skipped. */
int parac_gpu_download_times(parac_gpu_ctx* ctx, uint64_t* start_end);
/* TestHooks::on_phase (include/parac/factor_par.hpp:16-29, src/factor_par.cpp:112-120)
 * analogue of the last factor run with trace_phases set: dp[p*n + i] = the
 * dependency counter of position i as the eliminating warp/CTA read it at
 * phase p of trace_position's elimination (0 gathered, 1 sampled = after its
 * fill emissions, 2 decremented); taken[p] = 1 when phase p was reached
 * (a position with no merged entries stops after "gathered", as in the
 * reference). Counters of other positions may move concurrently, exactly as
 * under the reference's worker pool. */
int parac_gpu_download_phase_snapshots(parac_gpu_ctx* ctx, int64_t* dp, int32_t* taken);

/* Diagnostics: sub-phase timestamps sub[8*k + i] (then 4 rank-sort cycle counters per position at sub[8*n + 4*k]) of the same run (i = 0 setup
 * loads done, 1 gather landed, 2 weight sort done, 3 samples drawn, 4 fills
 * written, 5 release fence done; zero = not recorded on that path). */
int parac_gpu_download_subtimes(parac_gpu_ctx* ctx, uint64_t* sub);

/* Diagnostics: the cooperative hub path's per-column trace of the same
 * record_times run (kHubTraceWords = 64 words per wide column, layout in
 * csrc/cuda/factor_kernels.cuh). Copies min(cap, *count) records; *count =
 * wide columns recorded. */
int parac_gpu_download_hub_trace(parac_gpu_ctx* ctx, uint64_t* out, int32_t cap, int32_t* count);

/* Stage an existing factor (e.g. one computed by the reference) on the
 * device for the solve entry points. */
int parac_gpu_upload_factor(parac_gpu_ctx* ctx, int32_t n, const int64_t* col_ptr,
                            const int32_t* rows, const double* values, const double* diag,
                            const int32_t* perm);

/* schedule_levels (include/parac/factor_par.hpp:66, src/factor_par.cpp:659-684)
 * of the resident factor; returns the depth in *depth. levels may be NULL. */
int parac_gpu_schedule_levels(parac_gpu_ctx* ctx, int32_t* levels, int32_t* depth);

/* ordering_nnz_sort (ordering.hpp:32, src/ordering.cpp:49-70) on the device:
 * the same perm as parac_ordering_nnz_sort (bit-identical order: the fp64 tie
 * is an exact scaling of a 53-bit integer, so a stable radix sort by
 * (tie bits, degree) over vertices 0..n-1 reproduces std::sort's order).
 * Uses only g->ptr (degrees); does not touch the context's staged graph. */
int parac_gpu_ordering_nnz_sort(parac_gpu_ctx* ctx, const parac_csr* g, uint64_t seed, int32_t* perm);

/* ---- solve ------------------------------------------------------------------
 * SolveConfig / SolveReport (include/parac/solver.hpp:13-25). */
typedef struct {
  int32_t iterations;
  double relative_residual;   /* recomputed ||b - Lx|| / ||b|| */
  double recurrence_residual;
  int32_t converged;
  double solve_ms;            /* device time of the solve */
  double wall_ms;
  int32_t exact;              /* 1: the bit-exact PCG ran (every reduction, update and
                                 sweep in pcg_solve's order; x and the report are the
                                 reference's bytes), 0: the fast PCG */
} parac_gpu_solve_report;

/* pcg_solve (include/parac/solver.hpp:39-42, src/solver.cpp:95-175) on the
 * resident graph + factor. b, x are host arrays of length n (label space).
 * PARAC_NOT_CONNECTED for a disconnected graph, as the reference. */
int parac_gpu_pcg(parac_gpu_ctx* ctx, const double* b, double tol, int32_t max_iters, double* x,
                  parac_gpu_solve_report* report);
/* Mode of the solve path on ctx:
 *   0 default: parac_gpu_apply_preconditioner bit-identical to the reference
 *     (solver.cpp:32-74 summation order); parac_gpu_pcg exact (bit-identical
 *     to pcg_solve) for n <= 16384 (PARAC_EXACT_PCG_N), fast above;
 *   1 exact for both (any n); 2 fast for both. The exact PCG runs pcg_solve's
 *   serial reductions as single-thread chains (O(n) latency per dot product).
 *   Fast mode sums each row of the sweeps and each dot product in a fixed
 *   (run-to-run identical) tree order: same operator, different rounding, far
 *   shorter critical path; iteration counts within 10% of the reference. */
int parac_gpu_set_preconditioner_mode(parac_gpu_ctx* ctx, int32_t mode);
/* apply_preconditioner (solver.hpp:30, src/solver.cpp:32-74) */
int parac_gpu_apply_preconditioner(parac_gpu_ctx* ctx, const double* r, double* z);
/* laplacian_apply (solver.hpp:33, src/solver.cpp:76-93) */
int parac_gpu_laplacian_apply(parac_gpu_ctx* ctx, const double* x, double* y);
/* make_rhs (solver.hpp:47, src/solver.cpp:177-193); host computation (libm),
 * mode 1 = random_projected, 2 = from_random_x. */
int parac_make_rhs(const parac_csr* g, int mode, uint64_t seed, double* out);

/* ---- misc ---------------------------------------------------------------- */
/* LdlFactor::checksum (src/factor.cpp:17-36), host. */
uint64_t parac_factor_checksum(int32_t n, const int64_t* col_ptr, const int32_t* rows,
                               const double* values, const double* diag);
/* Pinned host memory for fast H2D/D2H (cudaMallocHost). */
void* parac_host_alloc(size_t bytes);
void parac_host_free(void* p);
/* Count of this library's kernel launches since process start. */
int64_t parac_gpu_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* PARAC_GPU_H */
