// parac_gpu_shim.hpp -- the C++ face of the B200 backend, in the reference's
// own namespace and types (/root/reference/proj/include/parac/*.hpp), so a
// maintainer adds `--backend gpu` to run_factor (proj/tools/parac_cli.cpp:106-128)
// with one include and one call. Header-only; it needs the reference headers
// on the include path and links against libparac_gpu.so (C ABI, parac_gpu.h).
//
//   LdlFactor parac::factor_gpu(graph, ordering, seed, GpuOptions, FactorStats*)
//       same shape as factor_parallel_left (include/parac/factor_par.hpp:53-62);
//       result is LdlFactor::same_values-identical to factor_randomized.
//   std::pair<std::vector<double>, SolveReport>
//   parac::pcg_solve_gpu(graph, factor, b, SolveConfig)
//       same shape as pcg_solve (include/parac/solver.hpp:39-42).
//   parac::apply_preconditioner_gpu / laplacian_apply_gpu   (solver.hpp:30,33)
//
// Errors: the C ABI returns parac::Errc values; they are rethrown here as
// parac::Error(code, detail) exactly like the CPU backends throw
// (ArenaExhausted, QueueStall, NotConnected, DimensionMismatch, ...).
// No exception crosses the C boundary; no CPU fallback exists behind it.
//
// Contexts: every call on a device shares ONE cached device context (buffers
// sized by the largest problem seen, pinned staging, solve layouts), created
// on first use. Calls are thread-safe: calls on the same device serialise on
// the context's mutex, calls on different devices run concurrently
// (factor_par's "no global state" contract becomes "one session per device").
// release_gpu_sessions() frees them (e.g. before cudaDeviceReset).
#pragma once

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <span>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>
#if defined(__linux__)
#include <sys/mman.h>
#endif

#include "parac/error.hpp"
#include "parac/factor.hpp"
#include "parac/factor_seq.hpp"
#include "parac/graph.hpp"
#include "parac/ordering.hpp"
#include "parac/solver.hpp"
#include "parac_gpu.h"

namespace parac {

// ParOptions analogue (include/parac/factor_par.hpp:31-45). workers has no
// meaning on the device; arena_budget maps to the column arena, the fill
// pool budget is separate (fills live in their own 16-byte slot pool).
struct GpuOptions {
  int device = 0;
  Index arena_budget = -1;       // column arena entries; <0: default (grown on demand)
  Index fill_pool_budget = -1;   // overflow fill entries; <0: default (grown on demand)
  double watchdog_seconds = 60.0;
  bool record_vertex_times = false;
  bool verify = false;           // TestHooks::verify analogue (device-side checks)
  int delay_ns = 0;              // TestHooks::delay analogue (random __nanosleep)
};

namespace gpu_detail {

[[noreturn]] inline void rethrow(int code) {
  std::string msg = parac_gpu_last_error();
  // the C ABI message is "<ErrcName>: detail"; Error prepends the name itself
  const std::string name = parac_errc_name(code);
  if (msg.rfind(name + ": ", 0) == 0) msg = msg.substr(name.size() + 2);
  throw Error(static_cast<Errc>(code), msg);
}
inline void check(int rc) {
  if (rc != 0) rethrow(rc);
}

// One cached context per device (see the header comment). Never destroyed
// implicitly: at process exit the driver reclaims it.
constexpr int kMaxDevices = 64;
struct Session {
  std::mutex m;
  parac_gpu_ctx* ctx = nullptr;
  // shape (n, adjacency entries) and factor size of the last factorization:
  // the guess for sizing the next same-shape factor's outputs early
  std::int64_t last_n = -1, last_nnz = -1, last_z = 0;
  // the row pointer rebuilt for each call (kept: a fresh 17 MB vector per
  // 128^3 call paid its page faults every time)
  std::vector<std::int64_t> ptr;
};
inline Session& session(int device) {
  static Session sessions[kMaxDevices];
  return sessions[device];
}
struct Ctx {  // a locked lease of a device's context
  std::unique_lock<std::mutex> lock;
  parac_gpu_ctx* c = nullptr;
  Session* s = nullptr;
  parac_gpu_ctx* get() const { return c; }
};
inline Ctx make_ctx(int device) {
  if (device < 0 || device >= kMaxDevices) throw Error(Errc::internal_error, "device ordinal out of range");
  Session& s = session(device);
  std::unique_lock<std::mutex> lock(s.m);
  if (!s.ctx) check(parac_gpu_create(device, &s.ctx));
  return Ctx{std::move(lock), s.ctx, &s};
}

// Sizes an output vector for a download. The host cost of the drop-in path
// is dominated by first-touch page faults on fresh multi-MB vectors (~110 ms
// for the 300 MB of a 128^3 factor on the B200 host's VM): large outputs ask
// for transparent huge pages (512x fewer faults) before resize() touches them.
template <typename T>
void size_output(std::vector<T>& v, std::size_t count) {
  static_assert(std::is_trivially_copyable_v<T>);
  v.reserve(count);
#if defined(__linux__) && defined(MADV_HUGEPAGE)
  const std::size_t bytes = count * sizeof(T);
  constexpr std::uintptr_t kHuge = std::uintptr_t{2} << 20;
  if (bytes >= 8 * kHuge) {
    const auto p = reinterpret_cast<std::uintptr_t>(v.data());
    const std::uintptr_t a = (p + kHuge - 1) & ~(kHuge - 1), e = (p + bytes) & ~(kHuge - 1);
    if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);  // a hint; failure is harmless
  }
#endif
  // first touch in parallel (the kernel zeroes each page on its fault, one
  // core per fault): resize() then writes over resident pages
  const std::size_t bytes_all = count * sizeof(T);
  if (bytes_all >= (std::size_t{16} << 20)) {
    char* base = reinterpret_cast<char*>(v.data());
    const int nt = 4;
    std::thread th[nt];
    for (int i = 0; i < nt; ++i)
      th[i] = std::thread([base, bytes_all, i] {
        const std::size_t a = bytes_all * i / nt, b = bytes_all * (i + 1) / nt;
        for (std::size_t off = a & ~std::size_t{4095}; off < b; off += 4096) base[off < a ? a : off] = 0;
      });
    for (auto& t : th) t.join();
  }
  v.resize(count);
}

// LaplacianGraph keeps ptr_ private; its public spans are views into the
// contiguous adjacency arrays (graph.hpp:36-44), so the row pointer is rebuilt
// from degree() and the arrays are passed without copying.
struct CsrView {
  std::vector<std::int64_t>& ptr;
  parac_csr csr{};
  CsrView(const LaplacianGraph& g, std::vector<std::int64_t>& buf) : ptr(buf) {
    const VertexId n = g.num_vertices();
    ptr.resize(static_cast<std::size_t>(n) + 1, 0);
    // ptr[v] = offset of v's neighbour span in the contiguous adjacency
    // array: independent per vertex, so large graphs fill it on 4 threads
    const VertexId* base = n > 0 ? g.neighbors(0).data() : nullptr;
    auto fill = [&](VertexId a, VertexId b) {
      for (VertexId v = a; v < b; ++v) ptr[v] = static_cast<std::int64_t>(g.neighbors(v).data() - base);
    };
    if (n >= (1 << 20)) {
      constexpr int kParts = 8;
      std::thread th[kParts - 1];
      for (int i = 1; i < kParts; ++i)
        th[i - 1] = std::thread(fill, static_cast<VertexId>(static_cast<std::int64_t>(n) * i / kParts),
                                static_cast<VertexId>(static_cast<std::int64_t>(n) * (i + 1) / kParts));
      fill(0, static_cast<VertexId>(n / kParts));
      for (auto& t : th) t.join();
    } else {
      fill(0, n);
    }
    if (n > 0) ptr[n] = static_cast<std::int64_t>(g.nnz_off_diagonal());
    csr.n = n;
    csr.ptr = ptr.data();
    csr.adj = n > 0 ? g.neighbors(0).data() : nullptr;
    csr.w = n > 0 ? g.weights(0).data() : nullptr;
  }
};

inline void stage_factor(parac_gpu_ctx* ctx, const LdlFactor& f) {
  check(parac_gpu_upload_factor(ctx, f.n, f.col_ptr.data(), f.rows.data(), f.values.data(),
                                f.diag.data(), f.perm.data()));
}

}  // namespace gpu_detail

// Frees every cached device context (the next call creates a fresh one).
inline void release_gpu_sessions() {
  for (int d = 0; d < gpu_detail::kMaxDevices; ++d) {
    gpu_detail::Session& s = gpu_detail::session(d);
    std::lock_guard<std::mutex> lock(s.m);
    if (s.ctx) parac_gpu_destroy(s.ctx);
    s.ctx = nullptr;
  }
}

inline LdlFactor factor_gpu(const LaplacianGraph& graph, const Ordering& ordering,
                            std::uint64_t seed, const GpuOptions& options = {},
                            FactorStats* stats = nullptr) {
  using namespace gpu_detail;
  const auto start_time = std::chrono::steady_clock::now();
  const VertexId n = graph.num_vertices();
  if (ordering.size() != n)
    throw Error(Errc::dimension_mismatch, "ordering size does not match the graph");
  auto ctx = make_ctx(options.device);
  CsrView v(graph, ctx.s->ptr);
  parac_gpu_options o;
  parac_gpu_default_options(&o);
  o.column_arena_entries = options.arena_budget;
  o.fill_pool_entries = options.fill_pool_budget;
  o.watchdog_seconds = options.watchdog_seconds;
  o.record_stats = 1;
  o.verify = options.verify ? 1 : 0;
  o.delay_ns = options.delay_ns;
  o.record_times = options.record_vertex_times ? 1 : 0;
  parac_gpu_factor_info info{};
  const auto t_csr = std::chrono::steady_clock::now();
  // The output vectors are sized while the device works (their first-touch
  // page faults are the largest host cost): col_ptr and diag exactly,
  // rows/values at the size of the last factor of a graph of this shape
  // (corrected below when the guess is off).
  LdlFactor f;
  f.n = n;
  const std::int64_t nnz_adj = v.ptr.empty() ? 0 : v.ptr.back();
  Session& sess = *ctx.s;
  const std::size_t guess =
      sess.last_n == n && sess.last_nnz == nnz_adj ? static_cast<std::size_t>(sess.last_z) : 0;
  // The sizing (first-touch faults + the vectors' zero fill, ~20 ms of host
  // memory work at 128^3) starts first, on helper threads, and overlaps the
  // upload and the device work; parac_gpu_factor_end then copies the factor
  // out as its columns become final.
  std::thread sizer([&f, n, guess] {
    std::thread t2([&f, n] {
      size_output(f.col_ptr, static_cast<std::size_t>(n) + 1);
      size_output(f.diag, static_cast<std::size_t>(n));
    });
    if (guess) {
      std::thread t3([&f, guess] { size_output(f.rows, guess); });
      size_output(f.values, guess);
      t3.join();
    }
    t2.join();
  });
  int rc = parac_gpu_upload(ctx.get(), &v.csr, ordering.perm.data());
  if (rc == 0) rc = parac_gpu_factor_begin(ctx.get(), seed, &o);
  sizer.join();
  check(rc);
  const auto t_sized = std::chrono::steady_clock::now();
  rc = parac_gpu_factor_end(ctx.get(), &info, f.col_ptr.data(), guess ? f.rows.data() : nullptr,
                                      guess ? f.values.data() : nullptr, f.diag.data(),
                                      static_cast<std::int64_t>(guess));
  if (rc != 0 && rc != static_cast<int>(Errc::budget_exceeded)) check(rc);
  const auto t_fac = std::chrono::steady_clock::now();
  const auto z = static_cast<std::size_t>(info.nnz_off_diagonal);
  const bool refetch = !guess || z > guess;  // the guess was short: fetch rows/values now
  if (refetch) {
    size_output(f.rows, z);
    size_output(f.values, z);
  } else {
    f.rows.resize(z);
    f.values.resize(z);
  }
  sess.last_n = n;
  sess.last_nnz = nnz_adj;
  sess.last_z = static_cast<std::int64_t>(z);
  f.perm = ordering.perm;
  const auto t_alloc = std::chrono::steady_clock::now();
  std::vector<std::int32_t> md, se, fr;
  if (stats) {
    md.resize(n);
    se.resize(n);
    fr.resize(n);
  }
  if (refetch || stats)
    check(parac_gpu_download(ctx.get(), nullptr, refetch ? f.rows.data() : nullptr,
                             refetch ? f.values.data() : nullptr, nullptr, stats ? md.data() : nullptr,
                             stats ? se.data() : nullptr, stats ? fr.data() : nullptr));
  if (std::getenv("PARAC_SHIM_TIMING")) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t_end = std::chrono::steady_clock::now();
    std::fprintf(stderr,
                 "factor_gpu: csr %.2f ms | sizing || upload+begin %.2f ms | end (device %.2f ms, streamed download) "
                 "%.2f ms | outputs %.2f ms | rest %.2f ms\n",
                 ms(start_time, t_csr), ms(t_csr, t_sized), info.device_ms, ms(t_sized, t_fac), ms(t_fac, t_alloc),
                 ms(t_alloc, t_end));
  }
  if (stats) {
    stats->merged_degree = std::move(md);
    stats->samples_emitted = std::move(se);
    stats->fills_received = std::move(fr);
    stats->total_fills = info.total_fills;
    stats->arena_used = info.arena_used;
    if (options.record_vertex_times) {
      std::vector<std::uint64_t> t(8 * static_cast<std::size_t>(n));
      check(parac_gpu_download_times(ctx.get(), t.data()));
      std::uint64_t t0 = ~0ull;
      for (VertexId k = 0; k < n; ++k)
        if (t[8 * k] && t[8 * k] < t0) t0 = t[8 * k];
      stats->vertex_seconds.assign(n, 0.0);
      for (VertexId k = 0; k < n; ++k)
        if (t[8 * k + 7]) stats->vertex_seconds[k] = static_cast<double>(t[8 * k + 7] - t0) * 1e-9;
    }
    // wall clock at the API, like factor_sequential (src/factor_seq.cpp:46, :141-143):
    // upload, device factorization, download and the host vectors included
    stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - start_time).count();
  }
  return f;
}

// Many independent problems in one device pass (BASELINE config[4]); no
// reference counterpart (the reference loops over factor_randomized). Factor i
// is same_values-identical to factor_randomized(graphs[i], orderings[i], seeds[i]).
inline std::vector<LdlFactor> factor_batch_gpu(std::span<const LaplacianGraph> graphs,
                                               std::span<const Ordering> orderings,
                                               std::span<const std::uint64_t> seeds,
                                               const GpuOptions& options = {}) {
  using namespace gpu_detail;
  const std::size_t count = graphs.size();
  if (orderings.size() != count || seeds.size() != count || count == 0)
    throw Error(Errc::dimension_mismatch, "batch lists differ in length");
  auto ctx = make_ctx(options.device);
  std::vector<std::vector<std::int64_t>> ptrs(count);  // one row pointer per problem
  std::vector<CsrView> views;
  views.reserve(count);
  std::vector<parac_csr> csrs(count);
  std::vector<const std::int32_t*> perms(count);
  for (std::size_t i = 0; i < count; ++i) {
    if (orderings[i].size() != graphs[i].num_vertices())
      throw Error(Errc::dimension_mismatch, "ordering size does not match the graph");
    views.emplace_back(graphs[i], ptrs[i]);
    csrs[i] = views.back().csr;
    perms[i] = orderings[i].perm.data();
  }
  parac_gpu_options o;
  parac_gpu_default_options(&o);
  o.column_arena_entries = options.arena_budget;
  o.fill_pool_entries = options.fill_pool_budget;
  o.watchdog_seconds = options.watchdog_seconds;
  parac_gpu_factor_info info{};
  check(parac_gpu_factor_batch(ctx.get(), static_cast<std::int32_t>(count), csrs.data(), perms.data(),
                               seeds.data(), &o, &info));
  std::vector<LdlFactor> out(count);
  for (std::size_t i = 0; i < count; ++i) {
    std::int64_t z = 0;
    check(parac_gpu_batch_nnz(ctx.get(), static_cast<std::int32_t>(i), &z));
    LdlFactor& f = out[i];
    f.n = graphs[i].num_vertices();
    size_output(f.col_ptr, static_cast<std::size_t>(f.n) + 1);
    size_output(f.rows, static_cast<std::size_t>(z));
    size_output(f.values, static_cast<std::size_t>(z));
    size_output(f.diag, static_cast<std::size_t>(f.n));
    f.perm = orderings[i].perm;
    check(parac_gpu_download_batch(ctx.get(), static_cast<std::int32_t>(i), f.col_ptr.data(), f.rows.data(),
                                   f.values.data(), f.diag.data()));
  }
  return out;
}

inline std::pair<std::vector<double>, SolveReport> pcg_solve_gpu(const LaplacianGraph& graph,
                                                                 const LdlFactor& factor,
                                                                 std::span<const double> b,
                                                                 const SolveConfig& config = {},
                                                                 int device = 0) {
  using namespace gpu_detail;
  const VertexId n = graph.num_vertices();
  if (factor.n != n || static_cast<VertexId>(b.size()) != n)
    throw Error(Errc::dimension_mismatch, "graph, factor and rhs sizes differ");
  auto ctx = make_ctx(device);
  CsrView v(graph, ctx.s->ptr);
  check(parac_gpu_upload(ctx.get(), &v.csr, factor.perm.data()));
  stage_factor(ctx.get(), factor);
  std::vector<double> x(static_cast<std::size_t>(n));
  parac_gpu_solve_report r{};
  check(parac_gpu_pcg(ctx.get(), b.data(), config.tol, config.max_iters, x.data(), &r));
  SolveReport rep;
  rep.iterations = r.iterations;
  rep.relative_residual = r.relative_residual;
  rep.recurrence_residual = r.recurrence_residual;
  rep.converged = r.converged != 0;
  rep.solve_seconds = r.wall_ms * 1e-3;
  return {std::move(x), rep};
}

inline std::vector<double> apply_preconditioner_gpu(const LdlFactor& factor,
                                                    std::span<const double> r, int device = 0) {
  using namespace gpu_detail;
  if (static_cast<VertexId>(r.size()) != factor.n)
    throw Error(Errc::dimension_mismatch, "rhs size differs from the factor");
  auto ctx = make_ctx(device);
  stage_factor(ctx.get(), factor);
  std::vector<double> z(r.size());
  check(parac_gpu_apply_preconditioner(ctx.get(), r.data(), z.data()));
  return z;
}

inline std::vector<double> laplacian_apply_gpu(const LaplacianGraph& graph,
                                               std::span<const double> x, int device = 0) {
  using namespace gpu_detail;
  if (static_cast<VertexId>(x.size()) != graph.num_vertices())
    throw Error(Errc::dimension_mismatch, "vector size differs from the graph");
  auto ctx = make_ctx(device);
  CsrView v(graph, ctx.s->ptr);
  std::vector<std::int32_t> ident(static_cast<std::size_t>(graph.num_vertices()));
  for (VertexId i = 0; i < graph.num_vertices(); ++i) ident[i] = i;
  check(parac_gpu_upload(ctx.get(), &v.csr, ident.data()));
  std::vector<double> y(x.size());
  check(parac_gpu_laplacian_apply(ctx.get(), x.data(), y.data()));
  return y;
}

}  // namespace parac
