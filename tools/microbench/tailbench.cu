// Micro-benchmark of the one-CTA tail sweep (tail4_kernel) on synthetic level
// structures: nlev levels of r rows x len entries, indices into earlier rows.
// Prints ns per level. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr tailbench.cu -o tailbench
#include <cstdio>
#include <vector>
#include <random>
#include "../../paper_2505_02977_b200/csrc/cuda/solve_kernels.cu"

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
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(flush, rep, 256 << 20);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        tail4_kernel<true><<<1, kTailThreads, kT4Smem>>>(nt, nlev, 0, dl, de, di, dv, ts, dinv, nullptr, x, lt);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
      }
      std::vector<unsigned long long> h(nlev);
      cudaMemcpy(h.data(), lt, 8 * nlev, cudaMemcpyDeviceToHost);
      printf("rows/level %2d len %3d: %d levels, kernel %.1f us, %.0f ns/level (%s)\n", r, len, nlev, best * 1e3,
             (h[nlev - 1] - h[0]) / double(nlev - 1), cudaGetErrorString(cudaGetLastError()));
      cudaFree(dl); cudaFree(de); cudaFree(di); cudaFree(dv); cudaFree(ts); cudaFree(dinv); cudaFree(x); cudaFree(lt); cudaFree(flush);
    }
  }
  return 0;
}
