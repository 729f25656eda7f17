// Host graph assembly shared by the generators (graph_host.cpp) and the
// Matrix Market reader (mm_io.cpp).
#pragma once
#include <cstdint>
#include <vector>

#include "../../../include/parac_gpu.h"

namespace parac_gpu {

struct Edge {
  std::int32_t a, b;
  double w;
};

// LaplacianGraph::from_edges (proj/src/graph.cpp:21-83) into a library-owned
// parac_graph; throws Failure{internal_error} on self-loops, non-positive
// weights, out-of-range endpoints and duplicate pairs, like the reference.
void build_graph(std::int32_t n, const std::vector<Edge>& edges, parac_graph* out);

}  // namespace parac_gpu
