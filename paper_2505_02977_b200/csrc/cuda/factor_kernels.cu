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
  int cnt = 0;
  const long long b = d.ptr[v], e = d.ptr[v + 1];
  for (long long t = b; t < e; ++t) cnt += d.perm[d.adj[t]] > p;
  d.fdeg[p] = cnt;
  d.dp[p] = static_cast<int>(e - b) - cnt;  // earlier_degree = initial dependency count
  d.fill_cnt[p] = 0;
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

// ---------------------------------------------------------------- K2
__global__ void initial_ready_kernel(FactorDev d) {
  if (d.ctrl->status != 0) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ready = p < d.n && d.dp[p] == 0;
  const bool big = ready && d.fdeg[p] > kSmallCap;  // no fills yet: R = forward degree
  publish(d, ready, big, p, lane_id());
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
  pos_count_kernel<<<(d.n + 255) / 256, 256, 0, s>>>(d);
  note_launches(1);
  cudaError_t e = launch_scan(d.fdeg, d.n, d.fwd_ptr, tile_scratch, s);
  if (e != cudaSuccess) return e;
  int dev = 0;
  cudaGetDevice(&dev);
  pos_fill_kernel<<<num_sms(dev) * 8, 256, 0, s>>>(d);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_initial_ready(const FactorDev& d, cudaStream_t s) {
  if (d.n == 0) return cudaSuccess;
  initial_ready_kernel<<<(d.n + 255) / 256, 256, 0, s>>>(d);
  note_launches(1);
  return cudaGetLastError();
}

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

}  // namespace parac_gpu
