// Micro-benchmark: hand-off latencies that bound the level-scheduled sweeps
// and the elimination critical path on B200.
//   pingpong_*   two CTAs on different SMs bounce a token N times (one-way
//                latency = total / 2N) with different publication protocols
//   grid_barrier all co-resident CTAs (148 x k) pass N sense-reversing
//                barriers (atomicAdd arrive + relaxed poll)
//   cluster_bar  barrier.cluster.arrive/wait in a 16-CTA cluster
//   cta_bar      __syncthreads of a 1024-thread CTA
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 sync.cu -o sync
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// mode 0: relaxed store / relaxed poll (value is the flag)
// mode 1: data store + fence.acq_rel + relaxed flag store / relaxed poll + fence
// mode 2: st.release / ld.acquire
// mode 3: data + atomicAdd flag after __threadfence / relaxed poll
__global__ void pingpong(int* flags, double* data, int iters, int mode, long long* out) {
  if (threadIdx.x != 0) return;
  const int me = blockIdx.x;  // 0 or 1
  int* mine = flags + 64 * me;
  int* other = flags + 64 * (1 - me);
  const unsigned long long t0 = gt();
  for (int i = 1; i <= iters; ++i) {
    if (me == 0) {
      // send i
      if (mode == 0) st_relaxed(mine, i);
      else if (mode == 1) { data[0] = i; asm volatile("fence.acq_rel.gpu;" ::: "memory"); st_relaxed(mine, i); }
      else if (mode == 2) { data[0] = i; st_release(mine, i); }
      else { data[0] = i; __threadfence(); atomicAdd(mine, 1); }
      // wait for echo
      if (mode == 2) { while (ld_acquire(other) < i) {} }
      else { while (ld_relaxed(other) < i) {} if (mode == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
    } else {
      if (mode == 2) { while (ld_acquire(other) < i) {} }
      else { while (ld_relaxed(other) < i) {} if (mode == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
      if (mode == 0) st_relaxed(mine, i);
      else if (mode == 1) { data[8] = i; asm volatile("fence.acq_rel.gpu;" ::: "memory"); st_relaxed(mine, i); }
      else if (mode == 2) { data[8] = i; st_release(mine, i); }
      else { data[8] = i; __threadfence(); atomicAdd(mine, 1); }
    }
  }
  if (me == 0) out[mode] = static_cast<long long>(gt() - t0);
}

__global__ void grid_barrier(int* count, int* sense, int iters, long long* out) {
  __shared__ int local_sense;
  if (threadIdx.x == 0) local_sense = 0;
  __syncthreads();
  const unsigned long long t0 = gt();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      local_sense ^= 1;
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      if (atomicAdd(count, 1) == gridDim.x - 1) {
        *count = 0;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        st_relaxed(sense, local_sense);
      } else {
        while (ld_relaxed(sense) != local_sense) {}
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[5] = static_cast<long long>(gt() - t0);
}

__global__ void coop_grid_sync(int iters, long long* out) {
  cg::grid_group g = cg::this_grid();
  const unsigned long long t0 = gt();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[6] = static_cast<long long>(gt() - t0);
}

__global__ void __cluster_dims__(16, 1, 1) cluster_bar(int iters, long long* out) {
  const unsigned long long t0 = gt();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[7] = static_cast<long long>(gt() - t0);
}

__global__ void __cluster_dims__(8, 1, 1) cluster_bar8(int iters, long long* out) {
  const unsigned long long t0 = gt();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[8] = static_cast<long long>(gt() - t0);
}

__global__ void cta_bar(int iters, long long* out) {
  const unsigned long long t0 = gt();
  for (int i = 0; i < iters; ++i) __syncthreads();
  if (threadIdx.x == 0) out[9] = static_cast<long long>(gt() - t0);
}

__global__ void nanosleep_res(long long* out) {
  unsigned long long t0 = gt();
  for (int i = 0; i < 100; ++i) __nanosleep(100);
  out[10] = static_cast<long long>(gt() - t0);
  t0 = gt();
  for (int i = 0; i < 100; ++i) __nanosleep(1000);
  out[11] = static_cast<long long>(gt() - t0);
}

int main() {
  int* flags; double* data; long long* out; int* cnt;
  cudaMalloc(&flags, 4096); cudaMalloc(&data, 1 << 20); cudaMalloc(&out, 256); cudaMalloc(&cnt, 1024);
  cudaMemset(out, 0, 256);
  const int N = 20000;
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(flags, 0, 4096);
    pingpong<<<2, 32>>>(flags, data, N, mode, out);
    cudaDeviceSynchronize();
  }
  const int M = 1000;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMemset(cnt, 0, 1024);
  grid_barrier<<<sms, 256>>>(cnt, cnt + 32, M, out);
  cudaDeviceSynchronize();
  void* args[] = {(void*)&M, (void*)&out};
  cudaLaunchCooperativeKernel((void*)coop_grid_sync, sms, 256, args, 0, 0);
  cudaDeviceSynchronize();
  cudaFuncSetAttribute(cluster_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cluster_bar<<<16, 256>>>(M, out);
  cudaError_t e16 = cudaDeviceSynchronize();
  cluster_bar8<<<8, 256>>>(M, out);
  cudaDeviceSynchronize();
  cta_bar<<<1, 1024>>>(M, out);
  nanosleep_res<<<1, 32>>>(out);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, out, 128, cudaMemcpyDeviceToHost);
  const char* names[4] = {"relaxed value-as-flag", "data+fence+relaxed flag / poll+fence",
                          "st.release / ld.acquire", "data+threadfence+atomicAdd / relaxed poll"};
  for (int mode = 0; mode < 4; ++mode)
    printf("pingpong %-45s one-way %.0f ns\n", names[mode], (double)h[mode] / (2.0 * N));
  printf("grid barrier (%d CTAs, atomic+poll): %.0f ns\n", sms, (double)h[5] / M);
  printf("cooperative grid.sync (%d CTAs): %.0f ns\n", sms, (double)h[6] / M);
  printf("cluster barrier 16 CTAs: %.0f ns (%s)\n", (double)h[7] / M, cudaGetErrorString(e16));
  printf("cluster barrier 8 CTAs: %.0f ns\n", (double)h[8] / M);
  printf("__syncthreads 1024 thr: %.1f ns\n", (double)h[9] / M);
  printf("__nanosleep(100) %.0f ns, __nanosleep(1000) %.0f ns  (%s)\n", h[10] / 100.0, h[11] / 100.0,
         cudaGetErrorString(e));
  return 0;
}
