// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A flat C ABI over the UNMODIFIED reference library (parac, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// Python tests, the golden-fixture script and bench.py's reference arm call the
// reference's own public API:
//   LaplacianGraph::from_edges      proj/src/graph.cpp:21
//   gen_poisson3d / gen_random_*    proj/src/generators.cpp:14,110,136
//   ordering_random / nnz_sort      proj/src/ordering.cpp:38,49
//   factor_randomized / exact       proj/src/factor_seq.cpp:150,156
//   factor_parallel_left / right    proj/src/factor_par.cpp:632,643
//   schedule_levels / depth         proj/src/factor_par.cpp:659,686
//   apply_preconditioner / laplacian_apply / pcg_solve / make_rhs
//                                   proj/src/solver.cpp:32,76,95,177
//   read_laplacian / write_matrix_market / write_factor / read_factor /
//   write_vector / read_vector      proj/src/matrix_market.cpp:129-304
//   write_permutation / ordering_from_file  proj/src/ordering.cpp:72-93
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "parac/error.hpp"
#include "parac/factor.hpp"
#include "parac/factor_par.hpp"
#include "parac/factor_seq.hpp"
#include "parac/generators.hpp"
#include "parac/graph.hpp"
#include "parac/matrix_market.hpp"
#include "parac/ordering.hpp"
#include "parac/rng.hpp"
#include "parac/solver.hpp"

using namespace parac;

namespace {

thread_local std::string g_last_error;

struct FactorBox {
  LdlFactor f;
  FactorStats stats;
  bool has_stats = false;
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_last_error = e.what();
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return static_cast<int>(Errc::internal_error);
  }
}

Ordering ordering_from_perm(std::int32_t n, const std::int32_t* perm) {
  std::vector<VertexId> p(perm, perm + n);
  return Ordering::from_positions(std::move(p));
}

}  // namespace

extern "C" {

const char* pref_last_error() { return g_last_error.c_str(); }

double pref_unit_uniform(std::uint64_t seed, std::int64_t key, std::uint64_t counter) {
  return SampleStream::unit_uniform(seed, key, counter);
}
std::uint64_t pref_derive_seed(std::uint64_t seed, std::uint64_t salt) {
  return derive_seed(seed, salt);
}

// ---------------------------------------------------------------- graphs
int pref_graph_from_edges(std::int32_t n, std::int64_t m, const std::int32_t* a,
                          const std::int32_t* b, const double* w, void** out) {
  return guarded([&] {
    std::vector<Triplet> e(static_cast<std::size_t>(m));
    for (std::int64_t i = 0; i < m; ++i) e[static_cast<std::size_t>(i)] = {a[i], b[i], w[i]};
    *out = new LaplacianGraph(LaplacianGraph::from_edges(n, e));
  });
}

int pref_graph_poisson3d(std::int32_t n, int variant, double epsilon, double contrast,
                         std::uint64_t seed, void** out) {
  return guarded([&] {
    PoissonSpec s;
    s.n = n;
    s.variant = static_cast<PoissonVariant>(variant);
    s.epsilon = epsilon;
    s.contrast_ratio = contrast;
    s.seed = seed;
    s.budget_vertices = static_cast<Index>(1) << 40;
    *out = new LaplacianGraph(gen_poisson3d(s));
  });
}

int pref_graph_random_connected(std::int32_t n, std::int64_t extra, std::uint64_t seed,
                                int unit_weights, void** out) {
  return guarded([&] {
    *out = new LaplacianGraph(gen_random_connected(n, extra, seed, unit_weights != 0));
  });
}

int pref_graph_random_components(std::int32_t n, std::int32_t comps, std::int64_t extra,
                                 std::uint64_t seed, void** out) {
  return guarded([&] {
    *out = new LaplacianGraph(gen_random_components(n, comps, extra, seed));
  });
}

void pref_graph_free(void* g) { delete static_cast<LaplacianGraph*>(g); }

std::int32_t pref_graph_n(void* g) { return static_cast<LaplacianGraph*>(g)->num_vertices(); }
std::int64_t pref_graph_nnz(void* g) {
  return static_cast<LaplacianGraph*>(g)->nnz_off_diagonal();
}

// CSR export through the public accessors (ptr_ is private, graph.hpp:36-44).
void pref_graph_csr(void* gp, std::int64_t* ptr, std::int32_t* adj, double* w, double* wdeg) {
  const LaplacianGraph& g = *static_cast<LaplacianGraph*>(gp);
  ptr[0] = 0;
  for (VertexId v = 0; v < g.num_vertices(); ++v) {
    const auto nb = g.neighbors(v);
    const auto ww = g.weights(v);
    std::memcpy(adj + ptr[v], nb.data(), nb.size() * sizeof(std::int32_t));
    std::memcpy(w + ptr[v], ww.data(), ww.size() * sizeof(double));
    ptr[v + 1] = ptr[v] + static_cast<std::int64_t>(nb.size());
    if (wdeg) wdeg[v] = g.weighted_degree(v);
  }
}

int pref_connected_components(void* g, std::int32_t* label, std::int32_t* count) {
  return guarded([&] {
    ComponentInfo c = connected_components(*static_cast<LaplacianGraph*>(g));
    if (label) std::memcpy(label, c.label.data(), c.label.size() * sizeof(std::int32_t));
    *count = c.count;
  });
}

// ------------------------------------------------------------- orderings
int pref_ordering_random(std::int32_t n, std::uint64_t seed, std::int32_t* perm) {
  return guarded([&] {
    Ordering o = ordering_random(n, seed);
    std::memcpy(perm, o.perm.data(), o.perm.size() * sizeof(std::int32_t));
  });
}

int pref_ordering_nnz_sort(void* g, std::uint64_t seed, std::int32_t* perm) {
  return guarded([&] {
    Ordering o = ordering_nnz_sort(*static_cast<LaplacianGraph*>(g), seed);
    std::memcpy(perm, o.perm.data(), o.perm.size() * sizeof(std::int32_t));
  });
}

int pref_dependency_counts(void* g, const std::int32_t* perm, std::int32_t* out) {
  return guarded([&] {
    const LaplacianGraph& graph = *static_cast<LaplacianGraph*>(g);
    auto dp = dependency_counts(graph, ordering_from_perm(graph.num_vertices(), perm));
    std::memcpy(out, dp.data(), dp.size() * sizeof(std::int32_t));
  });
}

// --------------------------------------------------------------- factor
// backend: 0 = factor_randomized (seq), 1 = par-left, 2 = par-right, 3 = exact.
// wall_seconds = wall clock around the API call (host graph in, host factor
// out), the CPU timing rule of BASELINE.md §2.
int pref_factor(void* gp, const std::int32_t* perm, std::uint64_t seed, int backend,
                int workers, std::int64_t arena_budget, std::int64_t workspace_capacity,
                int want_stats, double* wall_seconds, void** out) {
  return guarded([&] {
    const LaplacianGraph& g = *static_cast<LaplacianGraph*>(gp);
    const Ordering o = ordering_from_perm(g.num_vertices(), perm);
    auto* box = new FactorBox;
    FactorStats* st = want_stats ? &box->stats : nullptr;
    box->has_stats = want_stats != 0;
    ParOptions po;
    po.workers = workers;
    po.arena_budget = arena_budget;
    po.workspace_capacity = workspace_capacity;
    const auto t0 = std::chrono::steady_clock::now();
    try {
      switch (backend) {
        case 0: box->f = factor_randomized(g, o, seed, st); break;
        case 1: box->f = factor_parallel_left(g, o, seed, po, st); break;
        case 2: box->f = factor_parallel_right(g, o, seed, po, st); break;
        case 3: box->f = factor_exact(g, o, st); break;
        default: throw Error(Errc::internal_error, "unknown backend");
      }
    } catch (...) {
      delete box;
      throw;
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (wall_seconds) *wall_seconds = std::chrono::duration<double>(t1 - t0).count();
    *out = box;
  });
}

// Star/centre dependency trace through TestHooks::on_phase
// (proj/include/parac/factor_par.hpp:16-29): snapshots of dp after the sampled
// and decremented phases of `vertex`. Returns the number of snapshots.
int pref_factor_left_trace(void* gp, const std::int32_t* perm, std::uint64_t seed,
                           int workers, std::int32_t vertex, std::int64_t* snaps,
                           int max_snaps, int* count, void** out) {
  return guarded([&] {
    const LaplacianGraph& g = *static_cast<LaplacianGraph*>(gp);
    const VertexId n = g.num_vertices();
    const Ordering o = ordering_from_perm(n, perm);
    int c = 0;
    TestHooks hooks;
    hooks.on_phase = [&](TestHooks::Phase ph, VertexId v, const std::vector<std::int64_t>& dp) {
      if (v == vertex && ph != TestHooks::Phase::gathered && c < max_snaps) {
        std::memcpy(snaps + static_cast<std::size_t>(c) * n, dp.data(), n * sizeof(std::int64_t));
        ++c;
      }
    };
    ParOptions po;
    po.workers = workers;
    po.hooks = &hooks;
    auto* box = new FactorBox;
    box->f = factor_parallel_left(g, o, seed, po, nullptr);
    *count = c;
    *out = box;
  });
}

void pref_factor_free(void* f) { delete static_cast<FactorBox*>(f); }

std::int32_t pref_factor_n(void* f) { return static_cast<FactorBox*>(f)->f.n; }
std::int64_t pref_factor_nnz_off(void* f) {
  return static_cast<FactorBox*>(f)->f.nnz_off_diagonal();
}

void pref_factor_copy(void* fp, std::int64_t* col_ptr, std::int32_t* rows, double* values,
                      double* diag, std::int32_t* perm) {
  const LdlFactor& f = static_cast<FactorBox*>(fp)->f;
  std::memcpy(col_ptr, f.col_ptr.data(), f.col_ptr.size() * sizeof(std::int64_t));
  std::memcpy(rows, f.rows.data(), f.rows.size() * sizeof(std::int32_t));
  std::memcpy(values, f.values.data(), f.values.size() * sizeof(double));
  std::memcpy(diag, f.diag.data(), f.diag.size() * sizeof(double));
  if (perm) std::memcpy(perm, f.perm.data(), f.perm.size() * sizeof(std::int32_t));
}

int pref_factor_stats(void* fp, std::int32_t* merged, std::int32_t* samples,
                      std::int32_t* fills, std::int64_t* total_fills, double* seconds) {
  auto* box = static_cast<FactorBox*>(fp);
  if (!box->has_stats) return -1;
  const FactorStats& s = box->stats;
  std::memcpy(merged, s.merged_degree.data(), s.merged_degree.size() * sizeof(std::int32_t));
  std::memcpy(samples, s.samples_emitted.data(), s.samples_emitted.size() * sizeof(std::int32_t));
  std::memcpy(fills, s.fills_received.data(), s.fills_received.size() * sizeof(std::int32_t));
  *total_fills = s.total_fills;
  *seconds = s.seconds;
  return 0;
}

std::uint64_t pref_factor_checksum(void* f) { return static_cast<FactorBox*>(f)->f.checksum(); }

int pref_factor_from_arrays(std::int32_t n, const std::int64_t* col_ptr,
                            const std::int32_t* rows, const double* values, const double* diag,
                            const std::int32_t* perm, void** out) {
  return guarded([&] {
    auto* box = new FactorBox;
    LdlFactor& f = box->f;
    f.n = n;
    f.col_ptr.assign(col_ptr, col_ptr + n + 1);
    f.rows.assign(rows, rows + col_ptr[n]);
    f.values.assign(values, values + col_ptr[n]);
    f.diag.assign(diag, diag + n);
    f.perm.assign(perm, perm + n);
    *out = box;
  });
}

int pref_schedule_levels(void* f, std::int32_t* levels) {
  return guarded([&] {
    auto l = schedule_levels(static_cast<FactorBox*>(f)->f);
    std::memcpy(levels, l.data(), l.size() * sizeof(std::int32_t));
  });
}

int pref_schedule_depth(void* f) { return schedule_depth(static_cast<FactorBox*>(f)->f); }

// --------------------------------------------------------------- solver
int pref_apply_preconditioner(void* f, const double* r, double* z) {
  return guarded([&] {
    const LdlFactor& fac = static_cast<FactorBox*>(f)->f;
    auto out = apply_preconditioner(fac, std::span<const double>(r, fac.n));
    std::memcpy(z, out.data(), out.size() * sizeof(double));
  });
}

int pref_laplacian_apply(void* g, const double* x, double* y) {
  return guarded([&] {
    const LaplacianGraph& graph = *static_cast<LaplacianGraph*>(g);
    auto out = laplacian_apply(graph, std::span<const double>(x, graph.num_vertices()));
    std::memcpy(y, out.data(), out.size() * sizeof(double));
  });
}

int pref_make_rhs(void* g, int mode, std::uint64_t seed, double* out) {
  return guarded([&] {
    auto v = make_rhs(*static_cast<LaplacianGraph*>(g), static_cast<RhsMode>(mode), seed);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}

int pref_pcg(void* g, void* f, const double* b, double tol, int max_iters, double* x,
             int* iterations, double* relres, double* recres, int* converged, double* seconds) {
  return guarded([&] {
    const LaplacianGraph& graph = *static_cast<LaplacianGraph*>(g);
    SolveConfig cfg;
    cfg.tol = tol;
    cfg.max_iters = max_iters;
    auto [xx, rep] = pcg_solve(graph, static_cast<FactorBox*>(f)->f,
                               std::span<const double>(b, graph.num_vertices()), cfg);
    std::memcpy(x, xx.data(), xx.size() * sizeof(double));
    *iterations = rep.iterations;
    *relres = rep.relative_residual;
    *recres = rep.recurrence_residual;
    *converged = rep.converged ? 1 : 0;
    *seconds = rep.solve_seconds;
  });
}


// ------------------------------------------------------------ Matrix Market
int pref_read_laplacian(const char* path, void** out) {
  return guarded([&] { *out = new LaplacianGraph(read_laplacian(path)); });
}
int pref_write_matrix_market(const char* path, void* g) {
  return guarded([&] { write_matrix_market(path, *static_cast<LaplacianGraph*>(g)); });
}
int pref_write_factor(void* f, const char* stem) {
  return guarded([&] { write_factor(static_cast<FactorBox*>(f)->f, stem); });
}
int pref_read_factor(const char* stem, const char* perm_path, void** out) {
  return guarded([&] {
    auto* box = new FactorBox;
    box->f = read_factor(stem, perm_path ? perm_path : "");
    *out = box;
  });
}
int pref_write_vector(const char* path, std::int64_t n, const double* v) {
  return guarded([&] { write_vector(path, std::span<const double>(v, static_cast<std::size_t>(n))); });
}
int pref_read_vector(const char* path, std::int64_t cap, double* v, std::int64_t* n) {
  return guarded([&] {
    auto x = read_vector(path);
    *n = static_cast<std::int64_t>(x.size());
    std::memcpy(v, x.data(), std::min<std::size_t>(x.size(), static_cast<std::size_t>(cap)) * sizeof(double));
  });
}
int pref_write_permutation(const char* path, std::int32_t n, const std::int32_t* perm) {
  return guarded([&] { write_permutation(path, ordering_from_perm(n, perm)); });
}
}  // extern "C"
