// Micro-benchmark: K3's CTA gather + merge of one column in isolation (one
// CTA, fills in the preallocated pool, data L2-resident after the first rep):
// cta_hash_merge (hash by row + per-run staging) vs the raw rank sort that
// precedes the run merge. clock64 around each, per R.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//          -I../../paper_2505_02977_b200/csrc/cuda hashmerge.cu -o hashmerge
#include <cstdio>
#include <vector>
#include <random>
#include "../../paper_2505_02977_b200/csrc/cuda/eliminate.cu"

namespace parac_gpu {
void note_launches(long long) {}
}
using namespace parac_gpu;

__global__ void bench(FactorDev d, int R, long long* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ CtaShared sh;
  char* smem = reinterpret_cast<char*>(smem_raw);
  if (threadIdx.x < kDirChunks) sh.dirrow[threadIdx.x] = 0;
  __syncthreads();
  const int P = next_pow2(R);
  long long th = 0, ts = 0;
  int m = 0;
  for (int rep = 0; rep < 6; ++rep) {
    Scratch S = carve(smem, kBigCap);
    __syncthreads();
    long long t0 = clock64();
    m = P <= kThreads ? cta_hash_merge<1>(d, 0, 0, 0, R, sh.dirrow, S, sh, nullptr)
        : P <= 2 * kThreads ? cta_hash_merge<2>(d, 0, 0, 0, R, sh.dirrow, S, sh, nullptr)
                            : cta_hash_merge<4>(d, 0, 0, 0, R, sh.dirrow, S, sh, nullptr);
    __syncthreads();
    long long t1 = clock64();
    if (P <= kThreads) cta_rank_raw<1>(d, 0, 0, 0, R, sh.dirrow, S, nullptr);
    else if (P <= 2 * kThreads) cta_rank_raw<2>(d, 0, 0, 0, R, sh.dirrow, S, nullptr);
    __syncthreads();
    long long t2 = clock64();
    if (rep >= 2) { th += t1 - t0; ts += t2 - t1; }
  }
  if (threadIdx.x == 0) { out[0] = th / 4; out[1] = ts / 4; out[2] = m; }
}

int main() {
  std::mt19937 rng(1);
  const int c0 = 1024;
  int4* pool; long long* out; Ctrl* ctrl;
  cudaMalloc(&pool, sizeof(int4) * c0);
  cudaMalloc(&out, 64);
  cudaMalloc(&ctrl, sizeof(Ctrl));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, kCtaSmem);
  for (int R : {8, 32, 100, 174, 256, 400, 512}) {
    const int rows = R * 10 / 17 + 1;  // ~1.7 entries per row, as on the 128^3 critical path
    std::vector<int4> h(c0);
    for (int s = 0; s < R; ++s) {
      const int row = 1000 + static_cast<int>(rng() % rows) * 37;
      const double w = 1.0 + (rng() % 1000) * 1e-3;
      long long wb; memcpy(&wb, &w, 8);
      h[s] = make_int4(row, 5000 + s, static_cast<int>(wb & 0xffffffff), static_cast<int>(wb >> 32));
    }
    cudaMemcpy(pool, h.data(), sizeof(int4) * c0, cudaMemcpyHostToDevice);
    FactorDev d{};
    d.pool0 = pool; d.c0 = c0; d.ctrl = ctrl;
    bench<<<1, kThreads, kCtaSmem>>>(d, R, out);
    long long o[3];
    cudaMemcpy(o, out, 24, cudaMemcpyDeviceToHost);
    printf("R=%4d m=%4lld  hash merge %6lld cyc | rank sort (no run merge) %6lld cyc\n", R, o[2], o[0], o[1]);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
