// Micro-benchmark of the one-CTA tail sweep (tail4_kernel) on synthetic level
// structures: nlev levels of r rows x len entries, indices into earlier rows.
// Prints ns per level. Build (after `make lib`; links the library's other objects):
//   B=../../paper_2505_02977_b200/build
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr tailbench.cu \
//     $B/capi.o $B/factor_kernels.o $B/eliminate.o $B/ordering.o $B/host_graph_host.o $B/host_mm_io.o -o tailbench
#include <cstdio>
#include <vector>
#include <random>
#include "../../paper_2505_02977_b200/csrc/cuda/solve_kernels.cu"


// floor experiments: a 1024-thread CTA doing only the per-level barriers (+ options)
template <int MODE>
__global__ void __launch_bounds__(1024, 1) floor_kernel(int nlev, const int* eidx, unsigned long long* lt, double* sink) {
  __shared__ double xs[1024];
  const int tid = threadIdx.x;
  xs[tid] = tid;
  __syncthreads();
  double acc = 0;
  for (int t = 0; t < nlev; ++t) {
    if (MODE == 1 && tid == 32) prefetch_l2(eidx + t * 64, 256);
    if (MODE == 2 && tid < 32) acc += eidx[(t + 2) * 32 + tid];
    if (tid < 32) acc += xs[(t + tid) & 1023];
    __syncthreads();
    if (tid == 0) xs[t & 1023] = acc;
    __syncthreads();
    if (MODE == 3 && tid == 0) lt[t] = globaltimer_ns();
  }
  if (tid == 0) sink[0] = acc;
}

int main() {
  using namespace parac_gpu;
  cudaFuncSetAttribute(tail4_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kT4Smem));
  for (int r : {1, 4, 16, 32}) {
    for (int len : {3, 100, 700}) {
      const int nlev = std::min(800, kT3Rows / r - 1);
      const int nt = nlev * r;
      std::vector<int> lvl(nlev + 1), ep(nt + 1), idx;
      std::vector<double> val;
      std::mt19937 rng(1);
      for (int t = 0; t <= nlev; ++t) lvl[t] = t * r;
      for (int i = 0; i < nt; ++i) {
        ep[i] = static_cast<int>(idx.size());
        const int L = i / r;
        for (int q = 0; q < len; ++q) {
          idx.push_back(L > 0 ? static_cast<int>(rng() % (L * r)) : 0);
          val.push_back(L > 0 ? 1e-3 : 0.0);
        }
      }
      ep[nt] = static_cast<int>(idx.size());
      int *dl, *de, *di; double *dv, *ts, *dinv, *x; unsigned long long* lt;
      cudaMalloc(&dl, 4 * (nlev + 1)); cudaMalloc(&de, 4 * (nt + 1));
      cudaMalloc(&di, 4 * idx.size()); cudaMalloc(&dv, 8 * val.size());
      cudaMalloc(&ts, 8 * nt); cudaMalloc(&dinv, 8 * nt); cudaMalloc(&x, 8 * nt); cudaMalloc(&lt, 8 * (nlev + 8));
      cudaMemcpy(dl, lvl.data(), 4 * (nlev + 1), cudaMemcpyHostToDevice);
      cudaMemcpy(de, ep.data(), 4 * (nt + 1), cudaMemcpyHostToDevice);
      cudaMemcpy(di, idx.data(), 4 * idx.size(), cudaMemcpyHostToDevice);
      cudaMemcpy(dv, val.data(), 8 * val.size(), cudaMemcpyHostToDevice);
      cudaMemset(ts, 0, 8 * nt);
      // flush L2 between runs so the entries come from HBM like in the solver
      char* flush; cudaMalloc(&flush, 256 << 20);
      int4* pcs; cudaMalloc(&pcs, sizeof(int4) * 32 * nlev);
      tail4_pieces_kernel<<<(nlev + 7) / 8, 256>>>(nlev, 1, dl, de, pcs);
      int2* lrg; cudaMalloc(&lrg, sizeof(int2) * (nlev + 1));
      tail4_range_kernel<<<(nlev + 255) / 256, 256>>>(nlev, pcs, lrg);
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(flush, rep, 256 << 20);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        tail4_kernel<true><<<1, kTailThreads, kT4Smem>>>(nt, nlev, 0, pcs, lrg, di, dv, ts, dinv, nullptr, x, lt);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
      }
      std::vector<unsigned long long> h(nlev);
      cudaMemcpy(h.data(), lt, 8 * nlev, cudaMemcpyDeviceToHost);
      printf("rows/level %2d len %3d: %d levels, kernel %.1f us, %.0f ns/level (%s)\n", r, len, nlev, best * 1e3,
             (h[nlev - 1] - h[0]) / double(nlev - 1), cudaGetErrorString(cudaGetLastError()));
      if (r == 1 && len == 100) {
        auto var = [&](auto kern, const char* name) {
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kT4Smem));
          cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
          cudaEventRecord(a);
          kern<<<1, kTailThreads, kT4Smem>>>(nt, nlev, 0, pcs, lrg, di, dv, ts, dinv, nullptr, x, lt);
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b);
          printf("   variant %-24s %.0f ns/level\n", name, ms * 1e6 / nlev);
        };
        var(tail4_kernel<true, 1>, "no L2 prefetch");
        var(tail4_kernel<true, 2>, "no cp.async ring");
        var(tail4_kernel<true, 4>, "no result store");
        var(tail4_kernel<true, 8>, "no entry loads");
        var(tail4_kernel<true, 15>, "none of these");
      }
      cudaFree(dl); cudaFree(de); cudaFree(di); cudaFree(dv); cudaFree(ts); cudaFree(dinv); cudaFree(x); cudaFree(lt); cudaFree(flush);
    }
  }
  {
    int* di; double* sink; unsigned long long* lt;
    cudaMalloc(&di, 4 << 20); cudaMemset(di, 0, 4 << 20); cudaMalloc(&sink, 8); cudaMalloc(&lt, 8 * 1000);
    auto run = [&](auto kern, const char* name) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      kern<<<1, 1024>>>(800, di, lt, sink);
      cudaEventRecord(a);
      kern<<<1, 1024>>>(800, di, lt, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("floor %-28s %.0f ns/level\n", name, ms * 1e6 / 800);
    };
    run(floor_kernel<0>, "2 x syncthreads");
    run(floor_kernel<1>, "+ L2 bulk prefetch");
    run(floor_kernel<2>, "+ global load (2 ahead)");
    run(floor_kernel<3>, "+ globaltimer store");
  }
  return 0;
}
