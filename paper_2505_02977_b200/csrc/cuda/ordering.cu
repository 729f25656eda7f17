// Device ordering_nnz_sort (proj/src/ordering.cpp:49-70).
//
// The reference sorts (degree, tie, vertex) with std::sort, where
// tie = SampleStream::unit_uniform(derive_seed(seed, kSaltTieBreak), v, 0)
// = (x >> 11) * 2^-53. That fp64 value is an exact scaling of the 53-bit
// integer x >> 11, so comparing ties equals comparing those integers, and the
// whole key is an integer tuple: a stable LSD radix sort of the vertices
// 0..n-1 by (tie bits, then degree) yields exactly the reference order (the
// vertex id breaks remaining ties through stability). When the largest degree
// fits in 11 bits the two keys pack into one 64-bit key and one sort suffices.
// Then perm[vertex at p] = p. The sort is the hand-written one in
// radix_sort.cuh.

#include <algorithm>
#include <string>

#include "../host/errors.hpp"
#include "common.cuh"
#include "factor_kernels.cuh"
#include "radix_sort.cuh"

namespace parac_gpu {
void note_launches(long long k);  // defined in capi.cu
namespace {

__device__ __forceinline__ unsigned long long tie_bits(std::uint64_t seed, long long v) {
  std::uint64_t x = seed + 0x9e3779b97f4a7c15ULL * (static_cast<std::uint64_t>(v) + 1);
  x = dev::mix64(x);
  x = dev::mix64(x ^ (0xd1b54a32d192ed03ULL * 1ULL));  // counter 0
  return x >> 11;
}

__global__ void nnz_keys_kernel(int n, const long long* ptr, std::uint64_t tie_seed, int packed,
                                unsigned long long* key, int* vert) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const long long d = ptr[v + 1] - ptr[v];
    const unsigned long long t = tie_bits(tie_seed, v);
    key[v] = packed ? (static_cast<unsigned long long>(d) << 53) | t : t;
    vert[v] = v;
  }
}

__global__ void max_degree_kernel(int n, const long long* ptr, long long* maxdeg) {
  long long local = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    local = max(local, ptr[v + 1] - ptr[v]);
  for (int o = 16; o > 0; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned long long*>(maxdeg), static_cast<unsigned long long>(local));
}

__global__ void degree_of_kernel(int n, const long long* ptr, const int* vert, unsigned int* deg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int v = vert[i];
    deg[i] = static_cast<unsigned int>(ptr[v + 1] - ptr[v]);
  }
}

__global__ void positions_kernel(int n, const int* vert, int* perm) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) perm[vert[p]] = p;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Failure{internal_error, std::string(what) + ": " + cudaGetErrorString(e)};
}

int bits_for(unsigned long long v) {
  int b = 0;
  while (b < 64 && (v >> b) != 0) ++b;
  return std::max(b, 1);
}

}  // namespace

// Largest vertex degree of a device CSR into *d_out (zeroed here).
void max_degree_device(int n, const long long* d_ptr, long long* d_out, cudaStream_t st, int sms) {
  cuda_check(cudaMemsetAsync(d_out, 0, sizeof(long long), st), "memset");
  if (n <= 0) return;
  max_degree_kernel<<<std::min((n + 255) / 256, sms * 8), 256, 0, st>>>(n, d_ptr, d_out);
  note_launches(1);
}

void nnz_sort_device(int n, const long long* d_ptr, std::uint64_t tie_seed, int* d_perm, cudaStream_t st, int sms) {
  if (n <= 0) return;
  const int grid = std::min((n + 255) / 256, sms * 8);
  long long* d_max = nullptr;
  cuda_check(cudaMallocAsync(&d_max, sizeof(long long), st), "alloc");
  cuda_check(cudaMemsetAsync(d_max, 0, sizeof(long long), st), "memset");
  max_degree_kernel<<<grid, 256, 0, st>>>(n, d_ptr, d_max);
  long long maxdeg = 0;
  cuda_check(cudaMemcpyAsync(&maxdeg, d_max, sizeof(long long), cudaMemcpyDeviceToHost, st), "d2h");
  cuda_check(cudaStreamSynchronize(st), "sync");
  const int dbits = bits_for(static_cast<unsigned long long>(maxdeg));
  const bool packed = dbits <= 11;
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  int *v0 = nullptr, *v1 = nullptr;
  const std::size_t N = static_cast<std::size_t>(n);
  cuda_check(cudaMallocAsync(&k0, N * 8, st), "alloc");
  cuda_check(cudaMallocAsync(&k1, N * 8, st), "alloc");
  cuda_check(cudaMallocAsync(&v0, N * 4, st), "alloc");
  cuda_check(cudaMallocAsync(&v1, N * 4, st), "alloc");
  nnz_keys_kernel<<<grid, 256, 0, st>>>(n, d_ptr, tie_seed, packed ? 1 : 0, k0, v0);
  note_launches(2);
  unsigned long long* kb[2] = {k0, k1};
  int* vb[2] = {v0, v1};
  const int end1 = packed ? 53 + dbits : 53;
  int cur = radix::sort_pairs(n, kb, vb, end1, st);
  if (!packed) {  // stable second pass by degree, u32 keys in the spare 64-bit key buffer
    unsigned int* d0 = reinterpret_cast<unsigned int*>(kb[cur ^ 1]);
    unsigned int* db[2] = {d0, d0 + N};  // the spare key buffer holds 2N u32
    int* vb2[2] = {vb[cur], vb[cur ^ 1]};
    degree_of_kernel<<<grid, 256, 0, st>>>(n, d_ptr, vb2[0], d0);
    note_launches(1);
    const int c2 = radix::sort_pairs(n, db, vb2, dbits, st);
    cur = vb2[c2] == v0 ? 0 : 1;
  }
  positions_kernel<<<grid, 256, 0, st>>>(n, vb[cur], d_perm);
  note_launches(1);
  for (void* p : {static_cast<void*>(k0), static_cast<void*>(k1), static_cast<void*>(v0), static_cast<void*>(v1),
                  static_cast<void*>(d_max)})
    cuda_check(cudaFreeAsync(p, st), "free");
}

}  // namespace parac_gpu
