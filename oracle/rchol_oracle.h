/* TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * Plain-C restatement of the reference's randomized approximate Cholesky
 * (parac, /root/reference/proj) and the PCG solve that consumes it. Used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * bit-exact oracle. Parity is PINNED: tests/test_oracle.py checks this file
 * against the reference's own known-answer tests (P3/K3/star, proj/tests/*)
 * and against golden vectors produced by the unmodified reference build
 * (oracle/_ref, tests/golden/make_golden.py).
 *
 * All indices after build_pos_graph are elimination POSITIONS.
 */
#ifndef RCHOL_ORACLE_H
#define RCHOL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.cpp:7-24 */
double   oracle_unit_uniform(uint64_t seed, int64_t key, uint64_t counter);
uint64_t oracle_derive_seed(uint64_t seed, uint64_t salt);

typedef struct {
  int32_t n;
  int64_t* col_ptr;   /* n+1 */
  int32_t* rows;      /* col_ptr[n] */
  double*  values;    /* col_ptr[n] */
  double*  diag;      /* n */
  int32_t* merged_degree;   /* n (FactorStats::merged_degree) */
  int32_t* samples_emitted; /* n */
  int32_t* fills_received;  /* n */
  int64_t  total_fills;
} oracle_factor;

/* Graph in label space: CSR with neighbours ascending (graph.hpp:55-59). */
/* Returns 0 or an Errc code (13 = dimension_mismatch). exact != 0 runs the
 * full-clique variant (factor_exact, factor_seq.cpp:117-129). */
int  oracle_factor_randomized(int32_t n, const int64_t* ptr, const int32_t* adj,
                              const double* w, const int32_t* perm, uint64_t seed,
                              int exact, oracle_factor* out);
void oracle_factor_free(oracle_factor* f);

/* build_pos_graph (factor_common.hpp:31-80); caller-allocated outputs, fwd_to /
 * fwd_w sized ptr[n]/2. */
void oracle_build_pos_graph(int32_t n, const int64_t* ptr, const int32_t* adj,
                            const double* w, const int32_t* perm, int64_t* fwd_ptr,
                            int32_t* fwd_to, double* fwd_w, int32_t* earlier_degree);

/* LdlFactor::checksum (factor.cpp:17-36) */
uint64_t oracle_checksum(int32_t n, const int64_t* col_ptr, const int32_t* rows,
                         const double* values, const double* diag);

/* schedule_levels (factor_par.cpp:659-684); returns depth. */
int32_t oracle_schedule_levels(int32_t n, const int64_t* col_ptr, const int32_t* rows,
                               int32_t* level);

/* solver.cpp:32-74, 76-93, 177-193 */
void oracle_apply_preconditioner(int32_t n, const int64_t* col_ptr, const int32_t* rows,
                                 const double* values, const double* diag,
                                 const int32_t* perm, const double* r, double* z);
void oracle_laplacian_apply(int32_t n, const int64_t* ptr, const int32_t* adj,
                            const double* w, const double* x, double* y);
void oracle_make_rhs(int32_t n, const int64_t* ptr, const int32_t* adj, const double* w,
                     int mode, uint64_t seed, double* out);

/* pcg_solve (solver.cpp:95-175). Returns 0 or Errc (14 = not_connected). */
int oracle_pcg(int32_t n, const int64_t* ptr, const int32_t* adj, const double* w,
               const int64_t* col_ptr, const int32_t* rows, const double* values,
               const double* diag, const int32_t* perm, const double* b, double tol,
               int max_iters, double* x, int* iterations, double* relres, double* recres,
               int* converged);

/* Harness generators (BASELINE configs 2D 5-point, 27-point, R-MAT): edge
 * lists (a < b, w) for LaplacianGraph::from_edges; kind 0 = poisson2d(size),
 * 1 = poisson27(size, seed), 2 = rmat(scale = size, ef 16, seed). Arrays are
 * malloc'd (free with oracle_free); returns the edge count. */
int64_t oracle_gen_edges(int kind, int32_t size, uint64_t seed, int32_t** a, int32_t** b,
                         double** w, int32_t* n);
void oracle_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
