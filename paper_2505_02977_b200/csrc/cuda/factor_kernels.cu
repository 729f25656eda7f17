// sm_100a kernels of the randomized approximate Cholesky factorization,
// setup and assembly side (the elimination kernel K3 is in eliminate.cu):
//
//   K1  pos_count_kernel / pos_fill_kernel  build_pos_graph (proj/src/factor_common.hpp:31-80)
//   K2  initial_ready_kernel                ParState ctor + publish_initial_ready
//                                           (proj/src/factor_par.cpp:144-183)
//   K4  assemble (scan + copy)              ParState::assemble (proj/src/factor_par.cpp:309-345)
#include "factor_device.cuh"
#include "factor_kernels.cuh"
#include "scan.cuh"

namespace parac_gpu {

void note_launches(long long k);  // defined in capi.cu

using namespace dev;
using namespace fdev;

namespace {

// ---------------------------------------------------------------- K1
// Thread per label v: position p = perm[v], forward degree (neighbours at later
// positions) and the initial dependency count earlier_degree[p]; also resets
// the per-position state of the elimination.
__global__ void pos_count_kernel(FactorDev d) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= d.n) return;
  const int p = d.perm[v];
  if (p < 0 || p >= d.n) {
    fail(d, kErrPerm, v);
    return;
  }
  if (atomicExch(&d.inv[p], v) != -1) fail(d, kErrPerm, v);
  const long long b = d.ptr[v], e = d.ptr[v + 1];
  if (e - b > kHeavyDeg) {
    // hub: counted and filled by a whole CTA (pos_*_heavy_kernel)
    d.heavy_list[atomicAdd(d.heavy_count, 1)] = v;
  } else {
    int cnt = 0;
    for (long long t = b; t < e; ++t) cnt += d.perm[d.adj[t]] > p;
    d.fdeg[p] = cnt;
    d.cnt[p] = static_cast<unsigned long long>(static_cast<unsigned>(static_cast<int>(e - b) - cnt));  // earlier_degree
  }
  d.queue[p] = -1;
  d.bqueue[p] = -1;
  d.samples[p] = 0;
  d.col_len[p] = 0;  // K4 stays in bounds even when an aborted run skipped p
  d.col_start[p] = 0;
  if (d.level) d.level[p] = 1;
}

// Warp per position: forward neighbours (q > p) in ascending position order.
__global__ void pos_fill_kernel(FactorDev d) {
  if (d.ctrl->status != 0) return;
  const int lane = lane_id();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = gw; p < d.n; p += nw) {
    const int v = d.inv[p];
    const long long b = d.ptr[v];
    const int deg = static_cast<int>(d.ptr[v + 1] - b);
    const long long out = d.fwd_ptr[p];
    if (deg > kHeavyDeg) continue;  // pos_fill_heavy_kernel
    if (deg <= 32) {
      int q = -1;
      double wt = 0.0;
      if (lane < deg) {
        q = __ldg(d.perm + __ldg(d.adj + b + lane));
        wt = __ldg(d.w + b + lane);
      }
      const bool keep = q > p;
      int rank = 0;
      for (int j = 0; j < deg; ++j) {
        const int qj = __shfl_sync(kFull, q, j);
        rank += (qj > p) & (qj < q);
      }
      if (keep) {
        d.fwd_to[out + rank] = q;
        d.fwd_w[out + rank] = wt;
      }
    } else {
      // Wide row: rank each kept neighbour against the whole row (L1-resident).
      for (int base = 0; base < deg; base += 32) {
        const int t = base + lane;
        int q = -1;
        double wt = 0.0;
        if (t < deg) {
          q = __ldg(d.perm + __ldg(d.adj + b + t));
          wt = __ldg(d.w + b + t);
        }
        int rank = 0;
        for (int j = 0; j < deg; ++j) {
          const int qj = __ldg(d.perm + __ldg(d.adj + b + j));
          rank += (qj > p) & (qj < q);
        }
        if (q > p) {
          d.fwd_to[out + rank] = q;
          d.fwd_w[out + rank] = wt;
        }
      }
    }
  }
}

// Hubs (degree > kHeavyDeg): one CTA per vertex. Count: block reduction.
// Fill: block compaction of the kept (q, w) pairs into the forward range,
// then a sort by q: 1024-entry tiles in shared memory (bitonic), then
// merge-path passes ping-ponging with the hub scratch at the same offsets.
constexpr int kHT = 256;
__global__ void __launch_bounds__(kHT) pos_count_heavy_kernel(FactorDev d) {
  __shared__ int red[kHT / 32];
  const int nh = *d.heavy_count;
  for (int h = blockIdx.x; h < nh; h += gridDim.x) {
    const int v = d.heavy_list[h];
    const int p = d.perm[v];
    const long long b = d.ptr[v], e = d.ptr[v + 1];
    int cnt = 0;
    for (long long t = b + threadIdx.x; t < e; t += kHT) cnt += d.perm[d.adj[t]] > p;
    cnt = warp_sum(cnt);
    if (lane_id() == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      int c = 0;
      for (int w = 0; w < kHT / 32; ++w) c += red[w];
      d.fdeg[p] = c;
      d.cnt[p] = static_cast<unsigned long long>(static_cast<unsigned>(static_cast<int>(e - b) - c));
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kHT) pos_fill_heavy_kernel(FactorDev d) {
  __shared__ int base_sh;
  __shared__ int skey[1024];
  __shared__ double sval[1024];
  const int nh = *d.heavy_count;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int h = blockIdx.x; h < nh; h += gridDim.x) {
    const int v = d.heavy_list[h];
    const int p = d.perm[v];
    const long long b = d.ptr[v], e = d.ptr[v + 1];
    const long long out = d.fwd_ptr[p];
    const int f = static_cast<int>(d.fwd_ptr[p + 1] - out);
    int* K = d.fwd_to + out;
    double* V = d.fwd_w + out;
    int* K2 = d.heavy_key + out;
    double* V2 = d.heavy_val + out;
    if (tid == 0) base_sh = 0;
    __syncthreads();
    for (long long t0 = b; t0 < e; t0 += kHT) {  // compaction (any order)
      const long long t = t0 + tid;
      int q = -1;
      double w = 0.0;
      if (t < e) {
        q = d.perm[d.adj[t]];
        w = d.w[t];
      }
      const bool keep = q > p;
      const unsigned m = __ballot_sync(kFull, keep);
      int at = 0;
      if (lane == 0 && m) at = atomicAdd(&base_sh, __popc(m));
      at = __shfl_sync(kFull, at, 0);
      if (keep) {
        const int o = at + __popc(m & ((1u << lane) - 1));
        K[o] = q;
        V[o] = w;
      }
    }
    __syncthreads();
    // tiles of 1024: bitonic in shared memory (keys are unique positions)
    for (int tb = 0; tb < f; tb += 1024) {
      const int cnt = min(1024, f - tb);
      int P = 1;
      while (P < cnt) P <<= 1;
      for (int i = tid; i < P; i += kHT) {
        skey[i] = i < cnt ? K[tb + i] : 0x7fffffff;
        sval[i] = i < cnt ? V[tb + i] : 0.0;
      }
      __syncthreads();
      for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int i = tid; i < (P >> 1); i += kHT) {
            const int a = ((i & ~(j - 1)) << 1) | (i & (j - 1));
            const int c = a + j;
            const int ka = skey[a], kc = skey[c];
            if ((ka > kc) == ((a & k) == 0)) {
              skey[a] = kc;
              skey[c] = ka;
              const double tv = sval[a];
              sval[a] = sval[c];
              sval[c] = tv;
            }
          }
          __syncthreads();
        }
      }
      for (int i = tid; i < cnt; i += kHT) {
        K[tb + i] = skey[i];
        V[tb + i] = sval[i];
      }
      __syncthreads();
    }
    // merge passes
    int *sk = K, *dk = K2;
    double *sv = V, *dv = V2;
    for (int run = 1024; run < f; run *= 2) {
      for (int bb = 0; bb < f; bb += 2 * run) {
        const int na = min(run, f - bb), nb = max(0, min(run, f - bb - run));
        const int tot = na + nb;
        const int per = (tot + kHT - 1) / kHT;
        const int d0 = min(tid * per, tot), d1 = min(d0 + per, tot);
        if (d0 >= d1) continue;
        const int* A = sk + bb;
        const int* B = sk + bb + na;
        int lo = max(0, d0 - nb), hi = min(d0, na);
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (B[d0 - 1 - mid] < A[mid]) hi = mid; else lo = mid + 1;
        }
        int i = lo, j = d0 - lo;
        for (int o = d0; o < d1; ++o) {
          const bool takeA = j >= nb || (i < na && A[i] < B[j]);
          if (takeA) {
            dk[bb + o] = A[i];
            dv[bb + o] = sv[bb + i];
            ++i;
          } else {
            dk[bb + o] = B[j];
            dv[bb + o] = sv[bb + na + j];
            ++j;
          }
        }
      }
      __syncthreads();
      int* tk = sk; sk = dk; dk = tk;
      double* tv = sv; sv = dv; dv = tv;
    }
    if (sk != K) {
      for (int i = tid; i < f; i += kHT) {
        K[i] = sk[i];
        V[i] = sv[i];
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K2
// The initial frontier is published in ascending position order (a
// deterministic compaction instead of warp-aggregated appends): the heads of
// the longest dependency chains tend to be the lowest positions (every chain
// climbs in position), and the FIFO serves them first.
constexpr int kReadyThreads = 1024;
constexpr int kReadyItems = 4;
constexpr int kReadyTile = kReadyThreads * kReadyItems;

__device__ __forceinline__ void ready_flags(const FactorDev& d, int p, int& m, int& b) {
  const bool ready = p < d.n && (d.cnt[p] & 0xffffffffull) == 0;
  const bool big = ready && d.fdeg[p] > d.small_cap;  // no fills yet: R = forward degree
  m = ready && !big;
  b = big;
}

// per tile: counts of main / big ready positions
__global__ void __launch_bounds__(kReadyThreads) ready_count_kernel(FactorDev d, long long* tile_cnt) {
  __shared__ long long smem[32];
  long long cm = 0, cb = 0;
#pragma unroll
  for (int i = 0; i < kReadyItems; ++i) {
    int m, b;
    ready_flags(d, blockIdx.x * kReadyTile + i * kReadyThreads + threadIdx.x, m, b);
    cm += m;
    cb += b;
  }
  long long tm, tb;
  block_exclusive_scan(cm, smem, &tm);
  block_exclusive_scan(cb, smem, &tb);
  if (threadIdx.x == 0) {
    tile_cnt[2 * blockIdx.x] = tm;
    tile_cnt[2 * blockIdx.x + 1] = tb;
  }
}

// one CTA: exclusive scan of the tile counts; queue tails
__global__ void ready_scan_kernel(FactorDev d, long long* tile_cnt, int tiles) {
  __shared__ long long smem[32];
  long long base_m = 0, base_b = 0;
  for (int t0 = 0; t0 < tiles; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    const long long vm = t < tiles ? tile_cnt[2 * t] : 0, vb = t < tiles ? tile_cnt[2 * t + 1] : 0;
    long long sm, sb;
    const long long om = block_exclusive_scan(vm, smem, &sm);
    const long long ob = block_exclusive_scan(vb, smem, &sb);
    if (t < tiles) {
      tile_cnt[2 * t] = base_m + om;
      tile_cnt[2 * t + 1] = base_b + ob;
    }
    base_m += sm;
    base_b += sb;
  }
  if (threadIdx.x == 0) {
    d.ctrl->q_tail = static_cast<int>(base_m);
    d.ctrl->b_tail = static_cast<int>(base_b);
  }
}

// each tile writes its ready positions in order at its offsets
__global__ void __launch_bounds__(kReadyThreads) ready_scatter_kernel(FactorDev d, const long long* tile_off) {
  __shared__ long long smem[32];
  long long om = tile_off[2 * blockIdx.x], ob = tile_off[2 * blockIdx.x + 1];
  // blocked layout: thread t owns positions base + t*kReadyItems .. + kReadyItems - 1
  const int p0 = blockIdx.x * kReadyTile + threadIdx.x * kReadyItems;
  int m[kReadyItems], b[kReadyItems];
  long long cm = 0, cb = 0;
#pragma unroll
  for (int i = 0; i < kReadyItems; ++i) {
    ready_flags(d, p0 + i, m[i], b[i]);
    cm += m[i];
    cb += b[i];
  }
  long long tm, tb;
  long long xm = block_exclusive_scan(cm, smem, &tm) + om;
  long long xb = block_exclusive_scan(cb, smem, &tb) + ob;
#pragma unroll
  for (int i = 0; i < kReadyItems; ++i) {
    if (m[i]) d.queue[xm++] = p0 + i;
    if (b[i]) d.bqueue[xb++] = p0 + i;
  }
}

// ---------------------------------------------------------------- K4
__global__ void assemble_copy_kernel(FactorDev d, const long long* col_ptr, int* rows, double* vals) {
  const int lane = lane_id();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int k = gw; k < d.n; k += nw) {
    const int len = d.col_len[k];
    const long long from = d.col_start[k], to = col_ptr[k];
    for (int t = lane; t < len; t += 32) {
      rows[to + t] = d.arena_rows[from + t];
      vals[to + t] = d.arena_vals[from + t];
    }
  }
}

__global__ void sum_samples_kernel(FactorDev d) {
  long long s = 0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < d.n; p += gridDim.x * blockDim.x)
    s += d.samples[p];
  s = warp_sum(s);
  if (lane_id() == 0 && s) atomicAdd(reinterpret_cast<unsigned long long*>(&d.ctrl->total_fills),
                                     static_cast<unsigned long long>(s));
}

int num_sms(int device) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return sms > 0 ? sms : 148;
}

}  // namespace

long long scan_tiles(long long n) { return (n + kScanTile - 1) / kScanTile; }

cudaError_t launch_scan(const int* in, long long n, long long* out, long long* tile_scratch,
                        cudaStream_t s) {
  const long long tiles = scan_tiles(n);
  if (tiles == 0) return cudaMemsetAsync(out, 0, sizeof(long long), s);
  scan_tile_sums<<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, n, tile_scratch);
  scan_tile_offsets<<<1, 1024, 0, s>>>(tile_scratch, tiles);
  scan_finish<<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, n, tile_scratch, out);
  note_launches(3);
  return cudaGetLastError();
}

cudaError_t launch_pos_graph(const FactorDev& d, long long* tile_scratch, cudaStream_t s) {
  if (d.n == 0) return cudaSuccess;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e = cudaMemsetAsync(d.heavy_count, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  pos_count_kernel<<<(d.n + 255) / 256, 256, 0, s>>>(d);
  pos_count_heavy_kernel<<<num_sms(dev) * 4, kHT, 0, s>>>(d);
  note_launches(2);
  e = launch_scan(d.fdeg, d.n, d.fwd_ptr, tile_scratch, s);
  if (e != cudaSuccess) return e;
  pos_fill_kernel<<<num_sms(dev) * 8, 256, 0, s>>>(d);
  pos_fill_heavy_kernel<<<num_sms(dev) * 2, kHT, 0, s>>>(d);
  note_launches(2);
  return cudaGetLastError();
}

cudaError_t launch_initial_ready(const FactorDev& d, long long* tile_scratch, cudaStream_t s) {
  if (d.n == 0) return cudaSuccess;
  const int tiles = (d.n + kReadyTile - 1) / kReadyTile;
  ready_count_kernel<<<tiles, kReadyThreads, 0, s>>>(d, tile_scratch);
  ready_scan_kernel<<<1, 1024, 0, s>>>(d, tile_scratch, tiles);
  ready_scatter_kernel<<<tiles, kReadyThreads, 0, s>>>(d, tile_scratch);
  note_launches(3);
  return cudaGetLastError();
}
int initial_ready_scratch(int n) { return 2 * ((n + kReadyTile - 1) / kReadyTile) + 2; }

cudaError_t launch_assemble(const FactorDev& d, long long* col_ptr, int* rows, double* vals,
                            long long* tile_scratch, cudaStream_t s) {
  if (d.n == 0) return cudaMemsetAsync(col_ptr, 0, sizeof(long long), s);
  cudaError_t e = launch_scan(d.col_len, d.n, col_ptr, tile_scratch, s);
  if (e != cudaSuccess) return e;
  int dev = 0;
  cudaGetDevice(&dev);
  assemble_copy_kernel<<<num_sms(dev) * 8, 256, 0, s>>>(d, col_ptr, rows, vals);
  sum_samples_kernel<<<num_sms(dev) * 2, 256, 0, s>>>(d);
  note_launches(2);
  return cudaGetLastError();
}

cudaError_t launch_sum_samples(const FactorDev& d, cudaStream_t s) {
  if (d.n == 0) return cudaSuccess;
  int dev = 0;
  cudaGetDevice(&dev);
  sum_samples_kernel<<<num_sms(dev) * 2, 256, 0, s>>>(d);
  note_launches(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- batch
namespace {
__device__ __forceinline__ int batch_of(const long long* base, int count, long long x) {
  int lo = 0, hi = count - 1;  // last i with base[i] <= x
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (base[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}
__global__ void batch_vertex_kernel(int count, long long N, long long NNZ, const long long* base,
                                    const long long* ebase, long long* ptr, int* perm, int* pos_pid) {
  for (long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; j <= N;
       j += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (j == N) {
      ptr[N] = NNZ;
      continue;
    }
    const int i = batch_of(base, count, j);
    ptr[j] += ebase[i];
    perm[j] += static_cast<int>(base[i]);
    pos_pid[j] = i;  // positions of problem i are [base_i, base_{i+1}) too
  }
}
__global__ void batch_edge_kernel(int count, long long NNZ, const long long* ebase, const long long* base, int* adj) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < NNZ;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    adj[e] += static_cast<int>(base[batch_of(ebase, count, e)]);
}
__global__ void batch_rows_kernel(int n, const long long* col_ptr, const int* pos_pid, const long long* base,
                                  int* rows) {
  const int lane = lane_id();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int k = gw; k < n; k += nw) {
    const int b = static_cast<int>(base[pos_pid[k]]);
    for (long long t = col_ptr[k] + lane; t < col_ptr[k + 1]; t += 32) rows[t] -= b;
  }
}
}  // namespace

cudaError_t launch_batch_offsets(int count, long long N, long long NNZ, const long long* base,
                                 const long long* ebase, long long* ptr, int* adj, int* perm, int* pos_pid,
                                 cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  batch_vertex_kernel<<<num_sms(dev) * 8, 256, 0, s>>>(count, N, NNZ, base, ebase, ptr, perm, pos_pid);
  if (NNZ > 0) batch_edge_kernel<<<num_sms(dev) * 8, 256, 0, s>>>(count, NNZ, ebase, base, adj);
  note_launches(2);
  return cudaGetLastError();
}

namespace {
__global__ void extract_fills_kernel(int n, const unsigned long long* cnt, int* out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) out[p] = static_cast<int>(cnt[p] >> 32);
}
}  // namespace

cudaError_t launch_extract_fills(int n, const unsigned long long* cnt, int* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  extract_fills_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, cnt, out);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_batch_local_rows(int n, const long long* col_ptr, const int* pos_pid, const long long* base,
                                    int* rows, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  batch_rows_kernel<<<num_sms(dev) * 8, 256, 0, s>>>(n, col_ptr, pos_pid, base, rows);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace parac_gpu
