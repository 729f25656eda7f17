/* TEST INFRASTRUCTURE ONLY — see rchol_oracle.h. Each function cites the
 * reference file:line (paths relative to /root/reference/proj) it restates. */
#include "rchol_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng */
/* src/rng.cpp:7-11 */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* src/rng.cpp:15-20 */
double oracle_unit_uniform(uint64_t seed, int64_t key, uint64_t counter) {
  uint64_t x = seed + 0x9e3779b97f4a7c15ULL * ((uint64_t)key + 1);
  x = mix64(x);
  x = mix64(x ^ (0xd1b54a32d192ed03ULL * (counter + 1)));
  return (double)(x >> 11) * 0x1.0p-53;
}

/* src/rng.cpp:22-24 */
uint64_t oracle_derive_seed(uint64_t seed, uint64_t salt) { return mix64(seed ^ mix64(salt)); }

/* include/parac/rng.hpp:24 */
static const uint64_t kSaltSampling = 0x73616d706c696e67ULL;
static const uint64_t kSaltRhs = 0x7268735f76656320ULL;
/* src/factor_common.hpp:149 */
static const double kDropThreshold = 1e-300;

/* ------------------------------------------------------- pos graph (K1) */
typedef struct { int32_t q; double w; } qw_t;
static int cmp_qw(const void* a, const void* b) {
  const qw_t* x = (const qw_t*)a;
  const qw_t* y = (const qw_t*)b;
  /* std::pair<VertexId,double> ordering; q unique within a row */
  if (x->q != y->q) return x->q < y->q ? -1 : 1;
  return (x->w < y->w) ? -1 : (x->w > y->w);
}

/* src/factor_common.hpp:31-80 */
void oracle_build_pos_graph(int32_t n, const int64_t* ptr, const int32_t* adj,
                            const double* w, const int32_t* perm, int64_t* fwd_ptr,
                            int32_t* fwd_to, double* fwd_w, int32_t* earlier) {
  int32_t* inv = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  for (int32_t v = 0; v < n; ++v) inv[perm[v]] = v;
  memset(fwd_ptr, 0, sizeof(int64_t) * ((size_t)n + 1));
  memset(earlier, 0, sizeof(int32_t) * (size_t)n);
  for (int32_t v = 0; v < n; ++v) {
    const int32_t p = perm[v];
    for (int64_t t = ptr[v]; t < ptr[v + 1]; ++t) {
      if (perm[adj[t]] > p) ++fwd_ptr[p + 1]; else ++earlier[p];
    }
  }
  for (int32_t p = 0; p < n; ++p) fwd_ptr[p + 1] += fwd_ptr[p];
  qw_t* row = NULL;
  size_t row_cap = 0;
  for (int32_t p = 0; p < n; ++p) {
    const int32_t v = inv[p];
    size_t len = 0;
    const size_t deg = (size_t)(ptr[v + 1] - ptr[v]);
    if (deg > row_cap) { row_cap = deg * 2; row = (qw_t*)realloc(row, row_cap * sizeof(qw_t)); }
    for (int64_t t = ptr[v]; t < ptr[v + 1]; ++t) {
      const int32_t q = perm[adj[t]];
      if (q > p) { row[len].q = q; row[len].w = w[t]; ++len; }
    }
    qsort(row, len, sizeof(qw_t), cmp_qw);
    for (size_t i = 0; i < len; ++i) {
      fwd_to[fwd_ptr[p] + (int64_t)i] = row[i].q;
      fwd_w[fwd_ptr[p] + (int64_t)i] = row[i].w;
    }
  }
  free(row);
  free(inv);
}

/* ------------------------------------------------------------ factor */
/* RawEntry, src/factor_common.hpp:84-88 */
typedef struct { int32_t row; int32_t source; double weight; } raw_t;
/* MergedEntry, src/factor_common.hpp:90-94 */
typedef struct { int32_t row; int32_t mult; double weight; } merged_t;

typedef struct { raw_t* d; int32_t len, cap; } rawvec_t;

static void rawvec_push(rawvec_t* v, raw_t e) {
  if (v->len == v->cap) {
    v->cap = v->cap ? v->cap * 2 : 4;
    v->d = (raw_t*)realloc(v->d, sizeof(raw_t) * (size_t)v->cap);
  }
  v->d[v->len++] = e;
}

/* merge_raw sort key (row, source), src/factor_common.hpp:100-104 */
static int cmp_raw(const void* a, const void* b) {
  const raw_t* x = (const raw_t*)a;
  const raw_t* y = (const raw_t*)b;
  if (x->row != y->row) return x->row < y->row ? -1 : 1;
  return (x->source > y->source) - (x->source < y->source);
}

/* fill_sorted_view key (weight, row), src/factor_common.hpp:140-144 */
static int cmp_weight(const void* a, const void* b) {
  const merged_t* x = (const merged_t*)a;
  const merged_t* y = (const merged_t*)b;
  if (x->weight != y->weight) return x->weight < y->weight ? -1 : 1;
  return (x->row > y->row) - (x->row < y->row);
}

/* pick_by_suffix, include/parac/sampling.hpp:46-57 */
static size_t pick_by_suffix(const double* suffix, size_t lo, size_t hi, double u) {
  while (lo < hi) {
    size_t mid = lo + (hi - lo + 1) / 2;
    if (suffix[mid] > u) lo = mid; else hi = mid - 1;
  }
  return lo;
}

/* factor_sequential, src/factor_seq.cpp:43-146 (sampled: factor_randomized
 * :150-154; exact: factor_exact :156-159). */
int oracle_factor_randomized(int32_t n, const int64_t* ptr, const int32_t* adj,
                             const double* w, const int32_t* perm, uint64_t seed, int exact,
                             oracle_factor* out) {
  memset(out, 0, sizeof(*out));
  out->n = n;
  const int64_t nnz2 = ptr[n];
  int64_t* fwd_ptr = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
  int32_t* fwd_to = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz2 / 2 + 1));
  double* fwd_w = (double*)malloc(sizeof(double) * (size_t)(nnz2 / 2 + 1));
  int32_t* earlier = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  oracle_build_pos_graph(n, ptr, adj, w, perm, fwd_ptr, fwd_to, fwd_w, earlier);
  const uint64_t sample_seed = oracle_derive_seed(seed, kSaltSampling); /* :52 */

  rawvec_t* pending = (rawvec_t*)calloc((size_t)n + 1, sizeof(rawvec_t));
  out->col_ptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  out->diag = (double*)calloc((size_t)n + 1, sizeof(double));
  out->merged_degree = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  out->samples_emitted = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  out->fills_received = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  int64_t col_cap = nnz2 + 16, col_len = 0;
  out->rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)col_cap);
  out->values = (double*)malloc(sizeof(double) * (size_t)col_cap);

  rawvec_t raw = {0, 0, 0};
  merged_t* merged = NULL;
  double* suffix = NULL;
  int32_t mcap = 0;

  for (int32_t k = 0; k < n; ++k) {
    /* gather: forward edges (source -1) then pending fills, :71-84 */
    raw.len = 0;
    for (int64_t t = fwd_ptr[k]; t < fwd_ptr[k + 1]; ++t) {
      raw_t e = {fwd_to[t], -1, fwd_w[t]};
      rawvec_push(&raw, e);
    }
    rawvec_t* inc = &pending[k];
    out->fills_received[k] = inc->len;
    for (int32_t i = 0; i < inc->len; ++i) rawvec_push(&raw, inc->d[i]);
    free(inc->d);
    inc->d = NULL;
    inc->len = inc->cap = 0;

    /* merge_raw, src/factor_common.hpp:100-114 */
    qsort(raw.d, (size_t)raw.len, sizeof(raw_t), cmp_raw);
    if (raw.len > mcap) {
      mcap = raw.len * 2;
      merged = (merged_t*)realloc(merged, sizeof(merged_t) * (size_t)mcap);
      suffix = (double*)realloc(suffix, sizeof(double) * (size_t)mcap);
    }
    int32_t m = 0;
    for (int32_t i = 0; i < raw.len; ++i) {
      if (m > 0 && merged[m - 1].row == raw.d[i].row) {
        merged[m - 1].weight += raw.d[i].weight;
        merged[m - 1].mult += 1;
      } else {
        merged[m].row = raw.d[i].row;
        merged[m].weight = raw.d[i].weight;
        merged[m].mult = 1;
        ++m;
      }
    }
    out->col_ptr[k + 1] = out->col_ptr[k] + m; /* :87 */
    out->merged_degree[k] = m;
    if (m == 0) { out->diag[k] = 0.0; continue; } /* :92-95 */

    /* merged_total, src/factor_common.hpp:117-121 */
    double lkk = 0.0;
    for (int32_t i = 0; i < m; ++i) lkk += merged[i].weight;
    out->diag[k] = lkk;
    if (col_len + m > col_cap) {
      while (col_len + m > col_cap) col_cap *= 2;
      out->rows = (int32_t*)realloc(out->rows, sizeof(int32_t) * (size_t)col_cap);
      out->values = (double*)realloc(out->values, sizeof(double) * (size_t)col_cap);
    }
    for (int32_t i = 0; i < m; ++i) { /* :99-102 */
      out->rows[col_len] = merged[i].row;
      out->values[col_len] = -merged[i].weight / lkk;
      ++col_len;
    }

    int32_t emitted = 0;
#define PLACE_FILL(A, B, W)                                          \
    do {                                                             \
      const double w_ = (W);                                         \
      if (!(w_ < kDropThreshold)) {                                  \
        const int32_t lo_ = (A) < (B) ? (A) : (B);                   \
        const int32_t hi_ = (A) < (B) ? (B) : (A);                   \
        raw_t e_ = {hi_, k, w_};                                     \
        rawvec_push(&pending[lo_], e_);                              \
        ++emitted;                                                   \
      }                                                              \
    } while (0)
    if (!exact) {
      /* fill_sorted_view + sample_clique_sorted, sampling.hpp:66-84 */
      qsort(merged, (size_t)m, sizeof(merged_t), cmp_weight);
      if (m >= 2) {
        suffix[m - 1] = merged[m - 1].weight;
        for (int32_t g = m - 1; g-- > 0;) suffix[g] = merged[g].weight + suffix[g + 1];
        for (int32_t i = 0; i + 1 < m; ++i) {
          const double s = suffix[i + 1];
          const double u = oracle_unit_uniform(sample_seed, k, (uint64_t)i) * s;
          const size_t j = pick_by_suffix(suffix, (size_t)i + 1, (size_t)m - 1, u);
          const double wv = s * merged[i].weight / lkk;
          PLACE_FILL(merged[i].row, merged[j].row, wv);
        }
      }
    } else {
      /* full clique, src/factor_seq.cpp:117-129 */
      for (int32_t i = 0; i < m; ++i)
        for (int32_t j = i + 1; j < m; ++j)
          PLACE_FILL(merged[i].row, merged[j].row, merged[i].weight * merged[j].weight / lkk);
    }
#undef PLACE_FILL
    out->samples_emitted[k] = emitted;
    out->total_fills += emitted;
  }
  free(raw.d);
  free(merged);
  free(suffix);
  free(pending);
  free(fwd_ptr);
  free(fwd_to);
  free(fwd_w);
  free(earlier);
  return 0;
}

void oracle_factor_free(oracle_factor* f) {
  free(f->col_ptr);
  free(f->rows);
  free(f->values);
  free(f->diag);
  free(f->merged_degree);
  free(f->samples_emitted);
  free(f->fills_received);
  memset(f, 0, sizeof(*f));
}

/* ----------------------------------------------------------- checksum */
static uint64_t fnv1a(uint64_t h, const void* data, size_t bytes) {
  const unsigned char* p = (const unsigned char*)data;
  for (size_t i = 0; i < bytes; ++i) { h ^= p[i]; h *= 0x100000001b3ULL; }
  return h;
}

/* src/factor.cpp:17-36 */
uint64_t oracle_checksum(int32_t n, const int64_t* col_ptr, const int32_t* rows,
                         const double* values, const double* diag) {
  uint64_t h = 0xcbf29ce484222325ULL;
  h = fnv1a(h, &n, sizeof(n));
  h = fnv1a(h, col_ptr, ((size_t)n + 1) * sizeof(int64_t));
  h = fnv1a(h, rows, (size_t)col_ptr[n] * sizeof(int32_t));
  h = fnv1a(h, values, (size_t)col_ptr[n] * sizeof(double));
  h = fnv1a(h, diag, (size_t)n * sizeof(double));
  return h;
}

/* ----------------------------------------------------- schedule levels */
/* src/factor_par.cpp:659-691 */
int32_t oracle_schedule_levels(int32_t n, const int64_t* col_ptr, const int32_t* rows,
                               int32_t* level) {
  int32_t* blockers = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  int32_t* frontier = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  for (int64_t t = 0; t < col_ptr[n]; ++t) ++blockers[rows[t]];
  int32_t fl = 0, depth = 0;
  for (int32_t k = 0; k < n; ++k) { level[k] = 0; if (blockers[k] == 0) frontier[fl++] = k; }
  while (fl > 0) {
    ++depth;
    int32_t nl = 0;
    for (int32_t i = 0; i < fl; ++i) {
      const int32_t k = frontier[i];
      level[k] = depth;
      for (int64_t t = col_ptr[k]; t < col_ptr[k + 1]; ++t)
        if (--blockers[rows[t]] == 0) next[nl++] = rows[t];
    }
    int32_t* tmp = frontier; frontier = next; next = tmp;
    fl = nl;
  }
  free(blockers); free(frontier); free(next);
  return depth;
}

/* -------------------------------------------------------------- solver */
/* src/solver.cpp:32-74 */
void oracle_apply_preconditioner(int32_t n, const int64_t* col_ptr, const int32_t* rows,
                                 const double* values, const double* diag,
                                 const int32_t* perm, const double* r, double* z) {
  double* y = (double*)malloc(sizeof(double) * ((size_t)n + 1));
  for (int32_t v = 0; v < n; ++v) y[perm[v]] = r[v];
  for (int32_t k = 0; k < n; ++k) {
    const double yk = y[k];
    if (yk == 0.0) continue;
    for (int64_t p = col_ptr[k]; p < col_ptr[k + 1]; ++p) y[rows[p]] -= values[p] * yk;
  }
  for (int32_t k = 0; k < n; ++k) y[k] = diag[k] > 0.0 ? y[k] / diag[k] : 0.0;
  for (int32_t k = n; k-- > 0;) {
    double acc = y[k];
    for (int64_t p = col_ptr[k]; p < col_ptr[k + 1]; ++p) acc -= values[p] * y[rows[p]];
    y[k] = acc;
  }
  for (int32_t v = 0; v < n; ++v) z[v] = y[perm[v]];
  free(y);
}

/* wdeg as derived by LaplacianGraph::from_edges, src/graph.cpp:66-75 */
static double wdeg_of(const int64_t* ptr, const double* w, int32_t v) {
  double s = 0.0;
  for (int64_t t = ptr[v]; t < ptr[v + 1]; ++t) s += w[t];
  return s;
}

/* src/solver.cpp:76-93 */
void oracle_laplacian_apply(int32_t n, const int64_t* ptr, const int32_t* adj,
                            const double* w, const double* x, double* y) {
  for (int32_t v = 0; v < n; ++v) {
    double acc = wdeg_of(ptr, w, v) * x[v];
    for (int64_t t = ptr[v]; t < ptr[v + 1]; ++t) acc -= w[t] * x[adj[t]];
    y[v] = acc;
  }
}

/* src/solver.cpp:15-28 */
static double dotv(int32_t n, const double* a, const double* b) {
  double s = 0.0;
  for (int32_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static double norm2v(int32_t n, const double* a) { return sqrt(dotv(n, a, a)); }
static void subtract_mean(int32_t n, double* v) {
  double mean = 0.0;
  for (int32_t i = 0; i < n; ++i) mean += v[i];
  mean /= (double)n;
  for (int32_t i = 0; i < n; ++i) v[i] -= mean;
}

/* src/solver.cpp:177-193 (mode 1 random_projected, 2 from_random_x) */
void oracle_make_rhs(int32_t n, const int64_t* ptr, const int32_t* adj, const double* w,
                     int mode, uint64_t seed, double* out) {
  const uint64_t s = oracle_derive_seed(seed, kSaltRhs);
  double* v = (double*)malloc(sizeof(double) * ((size_t)n + 1));
  for (int32_t i = 0; i < n; ++i) {
    const double u1 = oracle_unit_uniform(s, i, 0);
    const double u2 = oracle_unit_uniform(s, i, 1);
    v[i] = sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586 * u2);
  }
  if (mode == 2) {
    oracle_laplacian_apply(n, ptr, adj, w, v, out);
  } else {
    subtract_mean(n, v);
    memcpy(out, v, sizeof(double) * (size_t)n);
  }
  free(v);
}

/* connected_components count, src/graph.cpp:188-210 */
static int32_t component_count(int32_t n, const int64_t* ptr, const int32_t* adj) {
  int32_t* label = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  int32_t* stack = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  for (int32_t i = 0; i < n; ++i) label[i] = -1;
  int32_t count = 0;
  for (int32_t s = 0; s < n; ++s) {
    if (label[s] != -1) continue;
    const int32_t id = count++;
    int32_t sp = 0;
    stack[sp++] = s;
    label[s] = id;
    while (sp > 0) {
      const int32_t v = stack[--sp];
      for (int64_t t = ptr[v]; t < ptr[v + 1]; ++t)
        if (label[adj[t]] == -1) { label[adj[t]] = id; stack[sp++] = adj[t]; }
    }
  }
  free(label); free(stack);
  return count;
}

/* src/solver.cpp:95-175 */
int oracle_pcg(int32_t n, const int64_t* ptr, const int32_t* adj, const double* w,
               const int64_t* col_ptr, const int32_t* rows, const double* values,
               const double* diag, const int32_t* perm, const double* b, double tol,
               int max_iters, double* x, int* iterations, double* relres, double* recres,
               int* converged) {
  if (component_count(n, ptr, adj) > 1) return 14; /* Errc::not_connected */
  const size_t bytes = sizeof(double) * ((size_t)n + 1);
  double* rhs = (double*)malloc(bytes);
  memcpy(rhs, b, sizeof(double) * (size_t)n);
  subtract_mean(n, rhs);
  const double b_norm = norm2v(n, rhs);
  for (int32_t i = 0; i < n; ++i) x[i] = 0.0;
  *iterations = 0; *relres = 0.0; *recres = 0.0; *converged = 0;
  if (b_norm == 0.0) { *converged = 1; free(rhs); return 0; }
  double* r = (double*)malloc(bytes);
  double* z = (double*)malloc(bytes);
  double* p = (double*)malloc(bytes);
  double* lp = (double*)malloc(bytes);
  double* best_x = (double*)malloc(bytes);
  memcpy(r, rhs, sizeof(double) * (size_t)n);
  oracle_apply_preconditioner(n, col_ptr, rows, values, diag, perm, r, z);
  memcpy(p, z, sizeof(double) * (size_t)n);
  double rz = dotv(n, r, z);
  memcpy(best_x, x, sizeof(double) * (size_t)n);
  double best_norm = norm2v(n, r);
  int iters = 0;
  while (iters < max_iters) {
    if (norm2v(n, r) <= tol * b_norm) break;
    ++iters;
    oracle_laplacian_apply(n, ptr, adj, w, p, lp);
    const double p_lp = dotv(n, p, lp);
    if (!(p_lp > 0.0)) break;
    const double alpha = rz / p_lp;
    for (int32_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * lp[i];
    }
    const double r_norm = norm2v(n, r);
    if (r_norm < best_norm) { best_norm = r_norm; memcpy(best_x, x, sizeof(double) * (size_t)n); }
    oracle_apply_preconditioner(n, col_ptr, rows, values, diag, perm, r, z);
    const double rz_next = dotv(n, r, z);
    const double beta = rz_next / rz;
    rz = rz_next;
    for (int32_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  double rec = norm2v(n, r);
  if (rec > best_norm) { memcpy(x, best_x, sizeof(double) * (size_t)n); rec = best_norm; }
  *recres = rec / b_norm;
  subtract_mean(n, x);
  oracle_laplacian_apply(n, ptr, adj, w, x, lp);
  for (int32_t i = 0; i < n; ++i) lp[i] = rhs[i] - lp[i];
  *iterations = iters;
  *relres = norm2v(n, lp) / b_norm;
  *converged = *relres <= tol;
  free(rhs); free(r); free(z); free(p); free(lp); free(best_x);
  return 0;
}

/* ------------------------------------------------- harness generators */
/* The BASELINE configs' synthetic inputs that the reference library has no
 * generator for (SURVEY §8(d) list items 1, 3, 4). They are harness
 * definitions, not reference code: the edge lists below are handed to the
 * reference's own LaplacianGraph::from_edges (src/graph.cpp:21) by the
 * reference arm of bench.py, so that arm never touches the product library.
 * tests/test_oracle.py pins the resulting CSR byte for byte to the product's
 * host generators. Weights of the form 0.5 + 1.5*U are computed with
 * -ffp-contract=off (FMA sensitivity). */
static const uint64_t kSaltCells = 0x63656c6c636f6566ULL;
static const uint64_t kSaltRmat = 0x726d61745f67656eULL;

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y ? 1 : 0;
}

int64_t oracle_gen_edges(int kind, int32_t size, uint64_t seed, int32_t** ea, int32_t** eb,
                         double** ew, int32_t* n_out) {
  int64_t cap = 0, m = 0;
  int32_t* A = NULL;
  int32_t* B = NULL;
  double* W = NULL;
  if (kind == 0) { /* 2D 5-point, id = x + N*y, unit weights */
    const int64_t N = size;
    cap = 2 * N * N;
    A = malloc(sizeof(int32_t) * cap); B = malloc(sizeof(int32_t) * cap); W = malloc(sizeof(double) * cap);
    for (int64_t y = 0; y < N; ++y)
      for (int64_t x = 0; x < N; ++x) {
        const int32_t v = (int32_t)(x + N * y);
        if (x + 1 < N) { A[m] = v; B[m] = v + 1; W[m] = 1.0; ++m; }
        if (y + 1 < N) { A[m] = v; B[m] = (int32_t)(v + N); W[m] = 1.0; ++m; }
      }
    *n_out = (int32_t)(N * N);
  } else if (kind == 1) { /* 3D 27-point, w(a,b) = 0.5 + 1.5 U(derive_seed(seed, cells), a, b), a < b */
    const int64_t N = size;
    const uint64_t ws = oracle_derive_seed(seed, kSaltCells);
    cap = 13 * N * N * N;
    A = malloc(sizeof(int32_t) * cap); B = malloc(sizeof(int32_t) * cap); W = malloc(sizeof(double) * cap);
    for (int64_t z = 0; z < N; ++z)
      for (int64_t y = 0; y < N; ++y)
        for (int64_t x = 0; x < N; ++x) {
          const int32_t a = (int32_t)(x + N * (y + N * z));
          for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
              for (int dx = -1; dx <= 1; ++dx) {
                const int64_t xx = x + dx, yy = y + dy, zz = z + dz;
                if (xx < 0 || yy < 0 || zz < 0 || xx >= N || yy >= N || zz >= N) continue;
                const int32_t b = (int32_t)(xx + N * (yy + N * zz));
                if (b <= a) continue;
                const double u = oracle_unit_uniform(ws, a, (uint64_t)b);
                const double t = 1.5 * u;
                A[m] = a; B[m] = b; W[m] = 0.5 + t; ++m;
              }
        }
    *n_out = (int32_t)(N * N * N);
  } else { /* R-MAT scale `size`, edge factor 16, Graph500 a,b,c = .57,.19,.19 */
    const int64_t nv = (int64_t)1 << size, samples = 16 * nv;
    const uint64_t rs = oracle_derive_seed(seed, kSaltRmat), ws = oracle_derive_seed(seed, kSaltCells);
    const double pa = 0.57, pb = 0.19, pc = 0.19;
    const double ab = pa + pb, abc = pa + pb + pc;
    uint64_t* keys = malloc(sizeof(uint64_t) * samples);
    for (int64_t e = 0; e < samples; ++e) {
      uint64_t u = 0, v = 0;
      for (int l = 0; l < size; ++l) {
        const double r = oracle_unit_uniform(rs, e, (uint64_t)l);
        const int bu = r >= ab;
        const int bv = (r >= pa && r < ab) || r >= abc;
        u = (u << 1) | (uint64_t)bu;
        v = (v << 1) | (uint64_t)bv;
      }
      keys[e] = u == v ? ~0ULL : ((u < v ? u : v) << 32) | (u < v ? v : u);
    }
    qsort(keys, (size_t)samples, sizeof(uint64_t), cmp_u64);
    cap = samples;
    A = malloc(sizeof(int32_t) * cap); B = malloc(sizeof(int32_t) * cap); W = malloc(sizeof(double) * cap);
    for (int64_t i = 0; i < samples; ++i) {
      if (keys[i] == ~0ULL) break;
      if (i > 0 && keys[i] == keys[i - 1]) continue;
      const int32_t a = (int32_t)(keys[i] >> 32), b = (int32_t)(keys[i] & 0xffffffffULL);
      const double t = 1.5 * oracle_unit_uniform(ws, a, (uint64_t)b);
      A[m] = a; B[m] = b; W[m] = 0.5 + t; ++m;
    }
    free(keys);
    *n_out = (int32_t)nv;
  }
  *ea = A; *eb = B; *ew = W;
  return m;
}

void oracle_free(void* p) { free(p); }
