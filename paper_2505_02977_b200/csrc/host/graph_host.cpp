// Host side of the boundary: graph construction, input generators and
// orderings, restating the reference's semantics so the device path sees the
// exact LaplacianGraph / Ordering the reference would build.
//   LaplacianGraph::from_edges   proj/src/graph.cpp:21-83
//   gen_poisson3d                proj/src/generators.cpp:14-65
//   gen_random_connected/components proj/src/generators.cpp:110-175
//   ordering_random / nnz_sort   proj/src/ordering.cpp:38-70
//   make_rhs                     proj/src/solver.cpp:177-193
//   LdlFactor::checksum          proj/src/factor.cpp:17-36
// Compiled with -ffp-contract=off and no -march (weights of the form
// 0.5 + 1.5*U change bits under FMA contraction).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <set>
#include <thread>
#include <vector>

#include "../../../include/parac_gpu.h"
#include "errors.hpp"
#include "graph_build.hpp"
#include "host_rng.hpp"

namespace parac_gpu {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

const char* errc_name(int code) {
  switch (code) {
    case 0: return "Ok";
    case asymmetric_input: return "AsymmetricInput";
    case positive_off_diagonal: return "PositiveOffDiagonal";
    case row_sum_violation: return "RowSumViolation";
    case too_large_for_dense: return "TooLargeForDense";
    case parse_error: return "ParseError";
    case unsupported_field: return "UnsupportedField";
    case budget_exceeded: return "BudgetExceeded";
    case not_a_permutation: return "NotAPermutation";
    case dense_blowup: return "DenseBlowup";
    case arena_exhausted: return "ArenaExhausted";
    case queue_stall: return "QueueStall";
    case workspace_full: return "WorkspaceFull";
    case dimension_mismatch: return "DimensionMismatch";
    case not_connected: return "NotConnected";
    case too_many_neighbors: return "TooManyNeighbors";
    case io_error: return "IoError";
    case internal_error: return "InternalError";
  }
  return "UnknownError";
}

namespace {

template <typename F>
void parallel_for(std::int64_t n, F&& f) {
  unsigned hw = std::thread::hardware_concurrency();
  if (hw == 0) hw = 1;
  const std::int64_t workers = std::min<std::int64_t>(hw, std::max<std::int64_t>(1, n / 65536));
  if (workers <= 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> pool;
  const std::int64_t chunk = (n + workers - 1) / workers;
  for (std::int64_t t = 0; t < workers; ++t) {
    const std::int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

template <typename T>
T* dup_array(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * std::max<std::size_t>(v.size(), 1)));
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

}  // namespace

// LaplacianGraph::from_edges, src/graph.cpp:21-83: place both halves in input
// order, sort each row by (neighbour, weight), reject duplicates, and sum the
// weighted degree left to right in ascending-neighbour order.
void build_graph(std::int32_t n, const std::vector<Edge>& edges, parac_graph* out) {
  std::vector<std::int64_t> ptr(static_cast<std::size_t>(n) + 1, 0);
  for (const Edge& e : edges) {
    if (e.a == e.b) throw Failure{internal_error, "self-loop edge " + std::to_string(e.a)};
    if (e.a < 0 || e.b < 0 || e.a >= n || e.b >= n)
      throw Failure{internal_error, "edge endpoint out of range"};
    if (!(e.w > 0.0))
      throw Failure{internal_error, "non-positive edge weight at (" + std::to_string(e.a) +
                                        ", " + std::to_string(e.b) + ")"};
    ++ptr[static_cast<std::size_t>(e.a) + 1];
    ++ptr[static_cast<std::size_t>(e.b) + 1];
  }
  for (std::int32_t v = 0; v < n; ++v) ptr[v + 1] += ptr[v];
  const std::int64_t nnz = ptr[n];
  std::vector<std::int32_t> adj(static_cast<std::size_t>(nnz));
  std::vector<double> w(static_cast<std::size_t>(nnz));
  {
    std::vector<std::int64_t> cursor(ptr.begin(), ptr.end() - 1);
    for (const Edge& e : edges) {
      std::int64_t at = cursor[e.a]++;
      adj[at] = e.b;
      w[at] = e.w;
      at = cursor[e.b]++;
      adj[at] = e.a;
      w[at] = e.w;
    }
  }
  std::vector<double> wdeg(static_cast<std::size_t>(n), 0.0);
  std::vector<std::int32_t> dup_row(1, -1);
  std::vector<std::int32_t> dup_col(1, -1);
  parallel_for(n, [&](std::int64_t lo, std::int64_t hi) {
    std::vector<std::pair<std::int32_t, double>> row;
    for (std::int64_t v = lo; v < hi; ++v) {
      row.clear();
      for (std::int64_t p = ptr[v]; p < ptr[v + 1]; ++p) row.emplace_back(adj[p], w[p]);
      std::sort(row.begin(), row.end());
      double sum = 0.0;
      for (std::size_t i = 0; i < row.size(); ++i) {
        if (i > 0 && row[i].first == row[i - 1].first) {
          dup_row[0] = static_cast<std::int32_t>(v);
          dup_col[0] = row[i].first;
        }
        adj[ptr[v] + static_cast<std::int64_t>(i)] = row[i].first;
        w[ptr[v] + static_cast<std::int64_t>(i)] = row[i].second;
        sum += row[i].second;
      }
      wdeg[v] = sum;
    }
  });
  if (dup_row[0] >= 0)
    throw Failure{internal_error, "duplicate edge (" + std::to_string(dup_row[0]) + ", " +
                                      std::to_string(dup_col[0]) + ")"};
  out->n = n;
  out->nnz = nnz;
  out->ptr = dup_array(ptr);
  out->adj = dup_array(adj);
  out->w = dup_array(w);
  out->wdeg = dup_array(wdeg);
}

namespace {

// LSD radix sort of 64-bit keys (used to dedupe R-MAT samples).
void radix_sort_u64(std::vector<std::uint64_t>& keys, int bits) {
  std::vector<std::uint64_t> tmp(keys.size());
  for (int shift = 0; shift < bits; shift += 11) {
    std::vector<std::size_t> count(2049, 0);
    for (std::uint64_t k : keys) ++count[((k >> shift) & 2047) + 1];
    for (int i = 0; i < 2048; ++i) count[i + 1] += count[i];
    for (std::uint64_t k : keys) tmp[count[(k >> shift) & 2047]++] = k;
    keys.swap(tmp);
  }
}

}  // namespace
}  // namespace parac_gpu

using namespace parac_gpu;

extern "C" {

const char* parac_errc_name(int code) { return errc_name(code); }
const char* parac_gpu_last_error(void) { return last_error(); }

void parac_graph_free(parac_graph* g) {
  if (!g) return;
  std::free(g->ptr);
  std::free(g->adj);
  std::free(g->w);
  std::free(g->wdeg);
  std::memset(g, 0, sizeof(*g));
}

int parac_graph_from_edges(int32_t n, int64_t m, const int32_t* a, const int32_t* b,
                           const double* w, parac_graph* out) {
  return guarded([&] {
    if (n < 0) throw Failure{internal_error, "negative vertex count"};
    std::vector<Edge> e(static_cast<std::size_t>(m));
    for (int64_t i = 0; i < m; ++i) e[static_cast<std::size_t>(i)] = {a[i], b[i], w[i]};
    build_graph(n, e, out);
  });
}

// gen_poisson3d, src/generators.cpp:14-65 (budget check omitted: the device
// path sizes itself from HBM, not the reference's 4M-vertex desk budget).
int parac_gen_poisson3d(int32_t n, int variant, double epsilon, double contrast_ratio,
                        uint64_t seed, parac_graph* out) {
  return guarded([&] {
    if (n < 2) throw Failure{budget_exceeded, "grid needs n >= 2"};
    if (epsilon <= 0.0 || contrast_ratio <= 0.0)
      throw Failure{parse_error, "epsilon and contrast ratio must be positive"};
    const std::int64_t N = n;
    const std::int64_t total = N * N * N;
    if (total > INT32_MAX) throw Failure{budget_exceeded, "grid exceeds int32 vertex ids"};
    auto vid = [N](std::int64_t x, std::int64_t y, std::int64_t z) {
      return static_cast<std::int32_t>(x + N * (y + N * z));
    };
    const std::uint64_t cell_seed = derive_seed(seed, kSaltCells);
    auto cell_coeff = [&](std::int32_t v) {
      const double u = unit_uniform(cell_seed, v, 0);
      return std::exp(u * std::log(contrast_ratio));
    };
    auto edge_weight = [&](std::int32_t a, std::int32_t b, bool z_dir) {
      switch (variant) {
        case 1: return z_dir ? epsilon : 1.0;
        case 2: {
          const double ca = cell_coeff(a);
          const double cb = cell_coeff(b);
          return 2.0 / (1.0 / ca + 1.0 / cb);
        }
        default: return 1.0;
      }
    };
    std::vector<Edge> edges;
    edges.reserve(static_cast<std::size_t>(3 * total));
    for (std::int64_t z = 0; z < N; ++z)
      for (std::int64_t y = 0; y < N; ++y)
        for (std::int64_t x = 0; x < N; ++x) {
          const std::int32_t v = vid(x, y, z);
          if (x + 1 < N) edges.push_back({v, vid(x + 1, y, z), edge_weight(v, vid(x + 1, y, z), false)});
          if (y + 1 < N) edges.push_back({v, vid(x, y + 1, z), edge_weight(v, vid(x, y + 1, z), false)});
          if (z + 1 < N) edges.push_back({v, vid(x, y, z + 1), edge_weight(v, vid(x, y, z + 1), true)});
        }
    build_graph(static_cast<std::int32_t>(total), edges, out);
  });
}

int parac_gen_poisson2d(int32_t n, parac_graph* out) {
  return guarded([&] {
    if (n < 2) throw Failure{budget_exceeded, "grid needs n >= 2"};
    const std::int64_t N = n;
    if (N * N > INT32_MAX) throw Failure{budget_exceeded, "grid exceeds int32 vertex ids"};
    std::vector<Edge> edges;
    edges.reserve(static_cast<std::size_t>(2 * N * N));
    for (std::int64_t y = 0; y < N; ++y)
      for (std::int64_t x = 0; x < N; ++x) {
        const auto v = static_cast<std::int32_t>(x + N * y);
        if (x + 1 < N) edges.push_back({v, static_cast<std::int32_t>(v + 1), 1.0});
        if (y + 1 < N) edges.push_back({v, static_cast<std::int32_t>(v + N), 1.0});
      }
    build_graph(static_cast<std::int32_t>(N * N), edges, out);
  });
}

int parac_gen_poisson27(int32_t n, uint64_t seed, parac_graph* out) {
  return guarded([&] {
    if (n < 2) throw Failure{budget_exceeded, "grid needs n >= 2"};
    const std::int64_t N = n;
    if (N * N * N > INT32_MAX) throw Failure{budget_exceeded, "grid exceeds int32 vertex ids"};
    const std::uint64_t ws = derive_seed(seed, kSaltCells);
    std::vector<Edge> edges;
    edges.reserve(static_cast<std::size_t>(13 * N * N * N));
    for (std::int64_t z = 0; z < N; ++z)
      for (std::int64_t y = 0; y < N; ++y)
        for (std::int64_t x = 0; x < N; ++x) {
          const auto a = static_cast<std::int32_t>(x + N * (y + N * z));
          for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
              for (int dx = -1; dx <= 1; ++dx) {
                const std::int64_t xx = x + dx, yy = y + dy, zz = z + dz;
                if (xx < 0 || yy < 0 || zz < 0 || xx >= N || yy >= N || zz >= N) continue;
                const auto b = static_cast<std::int32_t>(xx + N * (yy + N * zz));
                if (b <= a) continue;
                const double w = 0.5 + 1.5 * unit_uniform(ws, a, static_cast<std::uint64_t>(b));
                edges.push_back({a, b, w});
              }
        }
    build_graph(static_cast<std::int32_t>(N * N * N), edges, out);
  });
}

int parac_gen_rmat(int32_t scale, int32_t edge_factor, uint64_t seed, parac_graph* out) {
  return guarded([&] {
    if (scale < 1 || scale > 30) throw Failure{budget_exceeded, "rmat scale out of range"};
    const std::int64_t nv = std::int64_t{1} << scale;
    const std::int64_t samples = static_cast<std::int64_t>(edge_factor) * nv;
    const std::uint64_t rs = derive_seed(seed, kSaltRmat);
    const std::uint64_t ws = derive_seed(seed, kSaltCells);
    const double A = 0.57, B = 0.19, C = 0.19;
    std::vector<std::uint64_t> keys(static_cast<std::size_t>(samples));
    parallel_for(samples, [&](std::int64_t lo, std::int64_t hi) {
      for (std::int64_t e = lo; e < hi; ++e) {
        std::uint64_t u = 0, v = 0;
        for (int l = 0; l < scale; ++l) {
          const double r = unit_uniform(rs, e, static_cast<std::uint64_t>(l));
          const int bu = r >= A + B ? 1 : 0;
          const int bv = (r >= A && r < A + B) || r >= A + B + C ? 1 : 0;
          u = (u << 1) | static_cast<std::uint64_t>(bu);
          v = (v << 1) | static_cast<std::uint64_t>(bv);
        }
        if (u == v) {
          keys[e] = ~0ULL;
        } else {
          const std::uint64_t a = std::min(u, v), b = std::max(u, v);
          keys[e] = (a << 32) | b;
        }
      }
    });
    radix_sort_u64(keys, 64);
    std::vector<Edge> edges;
    edges.reserve(keys.size());
    for (std::size_t i = 0; i < keys.size(); ++i) {
      if (keys[i] == ~0ULL) break;
      if (i > 0 && keys[i] == keys[i - 1]) continue;
      const auto a = static_cast<std::int32_t>(keys[i] >> 32);
      const auto b = static_cast<std::int32_t>(keys[i] & 0xffffffffULL);
      edges.push_back({a, b, 0.5 + 1.5 * unit_uniform(ws, a, static_cast<std::uint64_t>(b))});
    }
    build_graph(static_cast<std::int32_t>(nv), edges, out);
  });
}

// src/generators.cpp:110-134
int parac_gen_random_connected(int32_t n, int64_t extra_edges, uint64_t seed, int unit_weights,
                               parac_graph* out) {
  return guarded([&] {
    SplitMix64 rng(derive_seed(seed, 0x67656e72616e64ULL));
    std::set<std::pair<std::int32_t, std::int32_t>> used;
    std::vector<Edge> edges;
    auto weight = [&]() { return unit_weights ? 1.0 : 0.5 + 1.5 * rng.next_double(); };
    for (std::int32_t v = 1; v < n; ++v) {
      const auto u = static_cast<std::int32_t>(rng.below(static_cast<std::uint64_t>(v)));
      used.emplace(u, v);
      edges.push_back({u, v, weight()});
    }
    const std::int64_t max_extra =
        static_cast<std::int64_t>(n) * (n - 1) / 2 - static_cast<std::int64_t>(edges.size());
    extra_edges = std::min(extra_edges, max_extra);
    while (extra_edges > 0) {
      auto a = static_cast<std::int32_t>(rng.below(static_cast<std::uint64_t>(n)));
      auto b = static_cast<std::int32_t>(rng.below(static_cast<std::uint64_t>(n)));
      if (a == b) continue;
      if (a > b) std::swap(a, b);
      if (!used.emplace(a, b).second) continue;
      edges.push_back({a, b, weight()});
      --extra_edges;
    }
    build_graph(n, edges, out);
  });
}

// src/generators.cpp:136-175
int parac_gen_random_components(int32_t n, int32_t components, int64_t extra_edges,
                                uint64_t seed, parac_graph* out) {
  return guarded([&] {
    components = std::max<std::int32_t>(1, std::min(components, n));
    SplitMix64 rng(derive_seed(seed, 0x636f6d706f6e74ULL));
    std::vector<Edge> edges;
    std::vector<std::int32_t> starts{0};
    for (std::int32_t c = 1; c < components; ++c)
      starts.push_back(static_cast<std::int32_t>(1 + rng.below(static_cast<std::uint64_t>(n - 1))));
    std::sort(starts.begin(), starts.end());
    starts.erase(std::unique(starts.begin(), starts.end()), starts.end());
    starts.push_back(n);
    std::set<std::pair<std::int32_t, std::int32_t>> used;
    for (std::size_t c = 0; c + 1 < starts.size(); ++c) {
      const std::int32_t lo = starts[c], hi = starts[c + 1];
      for (std::int32_t v = lo + 1; v < hi; ++v) {
        const std::int32_t u =
            lo + static_cast<std::int32_t>(rng.below(static_cast<std::uint64_t>(v - lo)));
        used.emplace(u, v);
        edges.push_back({u, v, 0.5 + 1.5 * rng.next_double()});
      }
      std::int64_t extras = extra_edges / static_cast<std::int64_t>(starts.size() - 1);
      const std::int32_t span = hi - lo;
      std::int64_t attempts = 8 * extras + 16;
      while (extras > 0 && span > 2 && attempts-- > 0) {
        auto a = lo + static_cast<std::int32_t>(rng.below(static_cast<std::uint64_t>(span)));
        auto b = lo + static_cast<std::int32_t>(rng.below(static_cast<std::uint64_t>(span)));
        if (a == b) continue;
        if (a > b) std::swap(a, b);
        if (!used.emplace(a, b).second) continue;
        edges.push_back({a, b, 0.5 + 1.5 * rng.next_double()});
        --extras;
      }
    }
    build_graph(n, edges, out);
  });
}

// src/ordering.cpp:38-47
int parac_ordering_random(int32_t n, uint64_t seed, int32_t* perm) {
  return guarded([&] {
    std::vector<std::int32_t> labels(static_cast<std::size_t>(n));
    std::iota(labels.begin(), labels.end(), 0);
    SplitMix64 rng(derive_seed(seed, kSaltOrdering));
    shuffle(labels, rng);
    for (std::int32_t p = 0; p < n; ++p) perm[labels[p]] = p;
  });
}

// src/ordering.cpp:49-70
int parac_ordering_nnz_sort(const parac_csr* g, uint64_t seed, int32_t* perm) {
  return guarded([&] {
    struct Key {
      std::int64_t degree;
      double tie;
      std::int32_t vertex;
    };
    const std::int32_t n = g->n;
    std::vector<Key> keys(static_cast<std::size_t>(n));
    const std::uint64_t tie_seed = derive_seed(seed, kSaltTieBreak);
    for (std::int32_t v = 0; v < n; ++v)
      keys[v] = {g->ptr[v + 1] - g->ptr[v], unit_uniform(tie_seed, v, 0), v};
    std::sort(keys.begin(), keys.end(), [](const Key& a, const Key& b) {
      if (a.degree != b.degree) return a.degree < b.degree;
      if (a.tie != b.tie) return a.tie < b.tie;
      return a.vertex < b.vertex;
    });
    for (std::int32_t p = 0; p < n; ++p) perm[keys[p].vertex] = p;
  });
}

// Ordering::from_positions, src/ordering.cpp:22-36
int parac_ordering_check(int32_t n, const int32_t* perm) {
  return guarded([&] {
    std::vector<std::uint8_t> seen(static_cast<std::size_t>(n), 0);
    for (std::int32_t v = 0; v < n; ++v) {
      const std::int32_t p = perm[v];
      if (p < 0 || p >= n || seen[p])
        throw Failure{not_a_permutation,
                      "position " + std::to_string(p) + " for vertex " + std::to_string(v)};
      seen[p] = 1;
    }
  });
}

// src/solver.cpp:177-193 (mode 1 random_projected, 2 from_random_x)
int parac_make_rhs(const parac_csr* g, int mode, uint64_t seed, double* out) {
  return guarded([&] {
    const std::int32_t n = g->n;
    std::vector<double> v(static_cast<std::size_t>(n));
    const std::uint64_t s = derive_seed(seed, kSaltRhs);
    for (std::int32_t i = 0; i < n; ++i) {
      const double u1 = unit_uniform(s, i, 0);
      const double u2 = unit_uniform(s, i, 1);
      v[i] = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586 * u2);
    }
    if (mode == 2) {
      for (std::int32_t r = 0; r < n; ++r) {
        double wd = 0.0;
        for (std::int64_t t = g->ptr[r]; t < g->ptr[r + 1]; ++t) wd += g->w[t];
        double acc = wd * v[r];
        for (std::int64_t t = g->ptr[r]; t < g->ptr[r + 1]; ++t) acc -= g->w[t] * v[g->adj[t]];
        out[r] = acc;
      }
      return;
    }
    double mean = 0.0;
    for (double x : v) mean += x;
    mean /= static_cast<double>(n);
    for (std::int32_t i = 0; i < n; ++i) out[i] = v[i] - mean;
  });
}

// src/factor.cpp:17-36
uint64_t parac_factor_checksum(int32_t n, const int64_t* col_ptr, const int32_t* rows,
                               const double* values, const double* diag) {
  auto fnv = [](std::uint64_t h, const void* data, std::size_t bytes) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (std::size_t i = 0; i < bytes; ++i) {
      h ^= p[i];
      h *= 0x100000001b3ULL;
    }
    return h;
  };
  std::uint64_t h = 0xcbf29ce484222325ULL;
  h = fnv(h, &n, sizeof(n));
  h = fnv(h, col_ptr, (static_cast<std::size_t>(n) + 1) * sizeof(std::int64_t));
  h = fnv(h, rows, static_cast<std::size_t>(col_ptr[n]) * sizeof(std::int32_t));
  h = fnv(h, values, static_cast<std::size_t>(col_ptr[n]) * sizeof(double));
  h = fnv(h, diag, static_cast<std::size_t>(n) * sizeof(double));
  return h;
}

}  // extern "C"
