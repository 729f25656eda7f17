// TEST INFRASTRUCTURE ONLY. Proves the drop-in: the reference's own types and
// API (compiled unmodified into oracle/_ref) side by side with the GPU backend
// through the C++ shim (paper_2505_02977_b200/csrc/shim/parac_gpu_shim.hpp),
// exactly as a `--backend gpu` branch of run_factor would call it.
//   factor_randomized (src/factor_seq.cpp:150)  vs  parac::factor_gpu
//   factor_parallel_left (src/factor_par.cpp:632) checksum vs the GPU's
//   pcg_solve (src/solver.cpp:95)               vs  parac::pcg_solve_gpu
//   Errc round trip: ArenaExhausted / DimensionMismatch / NotConnected
// Prints one line per check; exit code 0 only if all pass.
#include <cstdio>
#include <cstdlib>

#include "parac/factor_par.hpp"
#include "parac/generators.hpp"
#include "parac_gpu_shim.hpp"

using namespace parac;

static int failures = 0;
#define CHECK(cond, what)                                   \
  do {                                                      \
    const bool ok_ = (cond);                                \
    std::printf("%s %s\n", ok_ ? "PASS" : "FAIL", what);    \
    if (!ok_) ++failures;                                   \
  } while (0)

int main(int argc, char** argv) {
  const int side = argc > 1 ? std::atoi(argv[1]) : 32;
  PoissonSpec spec;
  spec.n = side;
  const LaplacianGraph g = gen_poisson3d(spec);
  const Ordering o = ordering_random(g.num_vertices(), 0);

  FactorStats st_ref, st_gpu;
  const LdlFactor ref = factor_randomized(g, o, 0, &st_ref);
  const LdlFactor gpu = factor_gpu(g, o, 0, GpuOptions{}, &st_gpu);
  CHECK(gpu.same_values(ref), "factor_gpu same_values factor_randomized");
  CHECK(gpu.checksum() == ref.checksum(), "checksum equal");
  CHECK(st_gpu.fills_received == st_ref.fills_received, "FactorStats::fills_received equal");
  CHECK(st_gpu.samples_emitted == st_ref.samples_emitted, "FactorStats::samples_emitted equal");
  CHECK(st_gpu.merged_degree == st_ref.merged_degree, "FactorStats::merged_degree equal");
  CHECK(st_gpu.total_fills == st_ref.total_fills, "FactorStats::total_fills equal");
  ParOptions po;
  po.workers = 4;
  const LdlFactor left = factor_parallel_left(g, o, 0, po);
  CHECK(left.checksum() == gpu.checksum(), "factor_parallel_left(w=4) checksum == GPU");

  const std::vector<double> b = make_rhs(g, RhsMode::random_projected, 0);
  SolveConfig cfg;
  cfg.tol = 1e-8;
  const auto [x_ref, rep_ref] = pcg_solve(g, ref, b, cfg);
  const auto [x_gpu, rep_gpu] = pcg_solve_gpu(g, gpu, b, cfg);
  std::printf("pcg iterations ref %d gpu %d, relres ref %.3e gpu %.3e\n", rep_ref.iterations,
              rep_gpu.iterations, rep_ref.relative_residual, rep_gpu.relative_residual);
  CHECK(rep_gpu.converged && rep_gpu.relative_residual <= cfg.tol, "pcg_solve_gpu converged to tol");
  CHECK(rep_gpu.iterations <= rep_ref.iterations + rep_ref.iterations / 10 &&
            rep_gpu.iterations >= rep_ref.iterations - rep_ref.iterations / 10,
        "pcg iterations within 10% of pcg_solve");

  const std::vector<double> z_ref = apply_preconditioner(ref, b);
  const std::vector<double> z_gpu = apply_preconditioner_gpu(gpu, b);
  CHECK(z_ref == z_gpu, "apply_preconditioner_gpu bit-identical");
  const std::vector<double> y_ref = laplacian_apply(g, b);
  const std::vector<double> y_gpu = laplacian_apply_gpu(g, b);
  CHECK(y_ref == y_gpu, "laplacian_apply_gpu bit-identical");

  // batch: three problems of different size/seed in one device pass
  {
    PoissonSpec s2;
    s2.n = side / 2 + 2;
    const LaplacianGraph g2 = gen_poisson3d(s2);
    const std::vector<LaplacianGraph> gs = {g, g2, g};
    const std::vector<Ordering> os = {o, ordering_random(g2.num_vertices(), 3), ordering_random(g.num_vertices(), 9)};
    const std::vector<std::uint64_t> ss = {0, 3, 9};
    const std::vector<LdlFactor> fb = factor_batch_gpu(gs, os, ss);
    bool all = fb.size() == 3;
    for (std::size_t i = 0; all && i < 3; ++i) all = fb[i].same_values(factor_randomized(gs[i], os[i], ss[i]));
    CHECK(all, "factor_batch_gpu: each problem same_values factor_randomized");
  }

  // error vocabulary: the same Errc codes the CPU backends throw
  try {
    GpuOptions tiny;
    tiny.arena_budget = 10;
    (void)factor_gpu(g, o, 0, tiny);
    CHECK(false, "ArenaExhausted thrown");
  } catch (const Error& e) {
    CHECK(e.code() == Errc::arena_exhausted, "ArenaExhausted thrown");
  }
  try {
    Ordering bad;
    bad.perm = {0, 1};
    (void)factor_gpu(g, bad, 0);
    CHECK(false, "DimensionMismatch thrown");
  } catch (const Error& e) {
    CHECK(e.code() == Errc::dimension_mismatch, "DimensionMismatch thrown");
  }
  try {
    const LaplacianGraph two = LaplacianGraph::from_edges(4, std::vector<Triplet>{{0, 1, 1.0}, {2, 3, 1.0}});
    const Ordering o2 = ordering_random(4, 0);
    const LdlFactor f2 = factor_gpu(two, o2, 0);
    (void)pcg_solve_gpu(two, f2, std::vector<double>{1, -1, 1, -1});
    CHECK(false, "NotConnected thrown");
  } catch (const Error& e) {
    CHECK(e.code() == Errc::not_connected, "NotConnected thrown");
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL PASS", failures);
  return failures ? 1 : 0;
}
