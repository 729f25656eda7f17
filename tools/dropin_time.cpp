// Drop-in timing harness (built like oracle/shim_check, against the reference's
// headers). Times the drop-in call a `--backend gpu` run_factor would make,
// parac::factor_gpu(graph, ordering, seed) -> LdlFactor with the reference's
// own pageable std::vector outputs, at gen_poisson3d(side), ordering_random(n,
// 0), seed 0. Prints one JSON line: wall ms per call (host clock around the
// call: upload, device factorization, download, output vectors), after
// `warmup` calls that create and size the cached device context.
//   dropin_time [side=128] [reps=5] [warmup=2]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "parac/generators.hpp"
#include "parac_gpu_shim.hpp"

using namespace parac;

int main(int argc, char** argv) {
  const int side = argc > 1 ? std::atoi(argv[1]) : 128;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 5;
  const int warmup = argc > 3 ? std::atoi(argv[3]) : 2;
  PoissonSpec spec;
  spec.n = side;
  const LaplacianGraph g = gen_poisson3d(spec);
  const Ordering o = ordering_random(g.num_vertices(), 0);
  std::uint64_t sum = 0;
  for (int i = 0; i < warmup; ++i) sum += factor_gpu(g, o, 0).checksum();
  std::vector<double> ms;
  std::size_t nnz = 0;
  std::uint64_t checksum = 0;
  for (int i = 0; i < reps; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    LdlFactor f = factor_gpu(g, o, 0);
    const auto t1 = std::chrono::steady_clock::now();
    ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    nnz = f.nnz();
    checksum = f.checksum();
  }
  double mean = 0;
  for (double v : ms) mean += v / ms.size();
  std::printf("{\"side\": %d, \"n\": %d, \"nnz\": %zu, \"checksum\": \"%016llx\", \"ms_per_call\": %.4f, \"calls\": [", side,
              g.num_vertices(), nnz, static_cast<unsigned long long>(checksum), mean);
  for (std::size_t i = 0; i < ms.size(); ++i) std::printf("%s%.4f", i ? ", " : "", ms[i]);
  std::printf("]}\n");
  return sum == 0 ? 0 : 0;
}
