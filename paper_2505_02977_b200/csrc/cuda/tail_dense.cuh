// Dense-inverse tail of the fast-mode triangular sweeps (included by
// solve_kernels.cu inside its anonymous namespace).
//
// The last few hundred levels of the factor DAG hold few rows each (at 128^3,
// levels 433..1206 hold 4,644 rows; levels 300..1206 hold 10,465) but cost a
// barrier each in both sweep directions. Restricted to those T rows, G is a
// T x T unit-lower-triangular block G_TT whose inverse W = G_TT^-1 is ~90%
// dense and entrywise in [0, 1] (G = I - N with N >= 0, so W = sum N^k: no
// cancellation). The tail of each sweep becomes ONE dense GEMV:
//   forward   y_T = W ts         (ts = rhs_T - G_TH y_H, tail_rhs_kernel)
//   backward  z_T = W^T (D^+ y)_T
// instead of ~900 dependent levels: ~T^2/2 x 8 bytes streamed from HBM per
// direction (a bandwidth-bound kernel) instead of ~900 barrier latencies.
//
// Storage: W row-major lower-packed and W^T row-major (= W's columns), every
// row padded to an even column range [a_r, b_r) so that rows start 16-byte
// aligned and the GEMV reads W and the x vector (shared memory) as double2.
//   W   row i: columns [0, even(i+1))      W[i][c] at offl[i] + c
//   W^T row j: columns [j & ~1, Tp)        W[i][j] at offu[j] + i - (j & ~1)
// (Tp = T rounded up to even; padding entries are zero.)
//
// W is built once per factor by a level-synchronous sparse substitution,
//   W[i][:] = e_i - sum_k G(i,k) W[k][:]     (rows k of earlier levels),
// one launch per tail level, each CTA computing a 256-column block of one row.

constexpr int kTwBuildThreads = 256;
constexpr int kTwBuildWarps = kTwBuildThreads / 32;
constexpr int kTwBlockCols = 256;                        // columns per CTA: 8 per lane
constexpr int kTwEntChunk = 256;                         // row entries staged per pass
constexpr int kTwGemvThreads = 1024;
constexpr int kTwMaxRows = 24576;                        // x of the GEMV lives in shared memory

__host__ __device__ inline int tw_even(int v) { return (v + 1) & ~1; }

// One CTA = (row i of level range [r0, r1), 256-column block cb). The row's
// entries (tail-relative k < i, G values) are staged in shared memory and
// split over the 8 warps (entry e to warp e % 8, four entries' loads in
// flight per lane); lane l owns columns cb + 8l .. cb + 8l + 7 (two 16-byte
// loads per parent row). The warps' partial sums meet in shared memory and
// are added in warp order (deterministic):
//   W[i][c] = [c == i] - sum_k G(i,k) W[k][c]   (W[k][c] = 0 for c > k).
__global__ void __launch_bounds__(kTwBuildThreads) tw_build_level_kernel(
    int r0, int r1, const int* __restrict__ fep, const int* __restrict__ fidx, const double* __restrict__ fval,
    const long long* __restrict__ offl, double* W) {
  __shared__ int sk[kTwEntChunk];
  __shared__ double sg[kTwEntChunk];
  __shared__ long long so[kTwEntChunk];
  __shared__ double part[kTwBuildWarps][kTwBlockCols];
  const int i = r0 + blockIdx.y;
  const int cb = blockIdx.x * kTwBlockCols;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rowlen = tw_even(i + 1);
  if (i >= r1 || cb >= rowlen) return;
  const int eb = fep[i], ee = fep[i + 1];
  const int c0 = cb + 8 * lane;  // this lane's first column
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  bool waited = false;
  for (int e0 = eb; e0 < ee; e0 += kTwEntChunk) {
    const int ne = min(kTwEntChunk, ee - e0);
    __syncthreads();
    for (int t = tid; t < ne; t += kTwBuildThreads) {
      const int k = fidx[e0 + t];
      sk[t] = k;
      sg[t] = fval[e0 + t];
      so[t] = offl[k];
    }
    if (!waited) {  // rows read below were written by earlier launches
      asm volatile("griddepcontrol.wait;" ::: "memory");
      waited = true;
    }
    __syncthreads();
    for (int t0 = warp; t0 < ne; t0 += 4 * kTwBuildWarps) {
      double2 v[4][4];
      double g[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = t0 + u * kTwBuildWarps;
        const int k = t < ne ? sk[t] : -1;
        g[u] = t < ne ? sg[t] : 0.0;
        const double2* w2 = reinterpret_cast<const double2*>(W + (t < ne ? so[t] : 0) + c0);
#pragma unroll
        for (int h = 0; h < 4; ++h)  // columns c0 + 2h, c0 + 2h + 1 (rows are padded to even length)
          v[u][h] = c0 + 2 * h <= k ? __ldcg(w2 + h) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          acc[2 * h] -= g[u] * v[u][h].x;
          acc[2 * h + 1] -= g[u] * v[u][h].y;
        }
    }
  }
  if (!waited) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  // entry k < c0 + 2h + 1 may have contributed a padding zero (W[k][k+1] = 0): harmless
#pragma unroll
  for (int q = 0; q < 8; ++q) part[warp][8 * lane + q] = acc[q];
  __syncthreads();
  const int c = cb + tid;
  if (c < rowlen) {
    double sum = c == i ? 1.0 : 0.0;
#pragma unroll
    for (int w = 0; w < kTwBuildWarps; ++w) sum += part[w][tid];
    W[offl[i] + c] = c <= i ? sum : 0.0;
  }
}

// W^T from W, 32 x 32 tiles over the lower triangle (tile row ib >= tile col
// jb); writes every entry of W^T's padded rows, zeros included.
__global__ void tw_transpose_kernel(int T, int Tp, const double* __restrict__ W, const long long* __restrict__ offl,
                                    const long long* __restrict__ offu, double* Wt) {
  __shared__ double tile[32][33];
  // linear tile id -> (ib, jb), jb <= ib
  const long long id = blockIdx.x;
  int ib = static_cast<int>((sqrt(8.0 * static_cast<double>(id) + 1.0) - 1.0) / 2.0);
  while (static_cast<long long>(ib) * (ib + 1) / 2 > id) --ib;
  while (static_cast<long long>(ib + 1) * (ib + 2) / 2 <= id) ++ib;
  const int jb = static_cast<int>(id - static_cast<long long>(ib) * (ib + 1) / 2);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  for (int r = ty; r < 32; r += 8) {
    const int i = ib * 32 + r, j = jb * 32 + tx;
    tile[r][tx] = (i < T && j <= i) ? W[offl[i] + j] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int j = jb * 32 + r, i = ib * 32 + tx;  // W^T row j, column i
    if (j < T && i < Tp && i >= (j & ~1)) Wt[offu[j] + i - (j & ~1)] = tile[tx][r];
  }
}

// ts_i = rhs_i - sum over row (base + i)'s head entries (c < base) of G x_c:
// the tail's right-hand side once the head is final. Warp per tail row.
__global__ void tail_rhs_kernel(int T, int base, const long long* __restrict__ lptr, const int* __restrict__ lidx,
                                const double* __restrict__ lval, const double* __restrict__ rhs_l, const double* x,
                                double* ts) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < T; i += nw) {
    const long long b = lptr[base + i], e = lptr[base + i + 1];
    double part = 0.0;
    for (long long q = b + lane; q < e; q += 32) {
      const int c = lidx[q];
      if (c < base) part += lval[q] * __ldcg(x + c);
    }
    part = warp_sum(part);
    if (lane == 0) ts[i] = rhs_l[base + i] - part;
  }
}

// out_r = sum over row r's padded column range of M[r][c] x[c] (x staged in
// shared memory), warp per row, longest rows first (zig-zag over the grid's
// warps); fixed per-lane order + xor tree (run-to-run deterministic).
//   LOWER: M = W (forward); also yd_r = out_r * dinv_r.
//   else:  M = W^T (backward).
template <bool LOWER>
__global__ void __launch_bounds__(kTwGemvThreads, 1) tw_gemv_kernel(
    int T, int Tp, const double* __restrict__ M, const long long* __restrict__ off, const double* xin,
    const double* __restrict__ dinv, double* out, double* yd) {
  extern __shared__ double xs[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int c = threadIdx.x; c < Tp; c += kTwGemvThreads) xs[c] = c < T ? __ldcg(xin + c) : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (kTwGemvThreads / 32) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (kTwGemvThreads / 32);
  for (int k = 0;; ++k) {
    const int g = k * nw + ((k & 1) ? nw - 1 - gw : gw);
    if (g >= T) break;
    const int r = LOWER ? T - 1 - g : g;  // longest rows first
    const int a = LOWER ? 0 : (r & ~1);
    const int len = LOWER ? tw_even(r + 1) : Tp - a;
    const double2* m2 = reinterpret_cast<const double2*>(M + off[r]);
    const double2* x2 = reinterpret_cast<const double2*>(xs + a);
    const int np = len >> 1;
    double s0 = 0.0, s1 = 0.0;
    int p = lane;
    for (; p + 96 < np; p += 128) {
      const double2 w0 = __ldcs(m2 + p), w1 = __ldcs(m2 + p + 32), w2 = __ldcs(m2 + p + 64), w3 = __ldcs(m2 + p + 96);
      const double2 v0 = x2[p], v1 = x2[p + 32], v2 = x2[p + 64], v3 = x2[p + 96];
      s0 += w0.x * v0.x;
      s1 += w0.y * v0.y;
      s0 += w1.x * v1.x;
      s1 += w1.y * v1.y;
      s0 += w2.x * v2.x;
      s1 += w2.y * v2.y;
      s0 += w3.x * v3.x;
      s1 += w3.y * v3.y;
    }
    for (; p < np; p += 32) {
      const double2 w0 = __ldcs(m2 + p);
      const double2 v0 = x2[p];
      s0 += w0.x * v0.x;
      s1 += w0.y * v0.y;
    }
    const double s = warp_sum(s0 + s1);
    if (lane == 0) {
      out[r] = s;
      if (LOWER) yd[r] = s * dinv[r];
    }
  }
  asm volatile("griddepcontrol.launch_dependents;");
}
