// hub.cu's hub_chains (lkk + suffix chains over global memory, staged) in
// isolation, one CTA, no other work on the SM (the chain section is a copy of
// hub.cu's).
#include <cstdio>
#include <cstdint>
constexpr int kThreads = 256;
__device__ __forceinline__ std::uint64_t globaltimer_ns() { std::uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__host__ __device__ __forceinline__ unsigned long long* hub_step(unsigned long long* rec, int p) { return rec + 8 + 4 * (p - 1); }
template <int U = 4, typename T>
__device__ __forceinline__ void stage_in(T* dst, const T* src, int cnt, int t, int nt, int stride = 1) {
  for (int i0 = t; i0 < cnt; i0 += U * nt) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { const int i = i0 + u * nt; if (i < cnt) v[u] = __ldcg(src + static_cast<long long>(i) * stride); }
#pragma unroll
    for (int u = 0; u < U; ++u) if (i0 + u * nt < cnt) dst[i0 + u * nt] = v[u];
  }
}
constexpr int kChainChunk = 512;

__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// s + x[0] + ... + x[cnt-1], left to right; the next 8 staged values load
// while the current 8 are added
__device__ __forceinline__ double chain_sum(double s, const double* x, int cnt) {
  int t = 0;
  if (cnt >= 8) {
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = x[q];
    for (t = 8; t + 8 <= cnt; t += 8) {
      double b[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) b[q] = x[t + q];
#pragma unroll
      for (int q = 0; q < 8; ++q) s = __dadd_rn(s, a[q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = b[q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) s = __dadd_rn(s, a[q]);
  }
  for (; t < cnt; ++t) s = __dadd_rn(s, x[t]);
  return s;
}

// o[g] = x[g] + (o[g+1] or the carried s), g = cnt-1 .. 0 (first chunk: the
// chain starts at x[cnt-1] itself). Returns the carried sum. The next 8
// values load before the current 8 are added and stored: with x and o both
// shared memory the compiler cannot move those loads above the stores itself
// (measured 12.3 -> ~9.5 cycles per element in isolation).
__device__ __forceinline__ double chain_suffix(double s, bool first, const double* x, double* o, int cnt) {
  int g = cnt - 1;
  if (first) {
    s = x[g];
    o[g] = s;
    --g;
  }
  if (g >= 7) {
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = x[g - q];
    for (; g - 15 >= 0; g -= 8) {
      double b[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) b[q] = x[g - 8 - q];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        s = __dadd_rn(a[q], s);
        o[g - q] = s;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = b[q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      s = __dadd_rn(a[q], s);
      o[g - q] = s;
    }
    g -= 8;
  }
  for (; g >= 0; --g) {
    s = __dadd_rn(x[g], s);
    o[g] = s;
  }
  return s;
}

// Returns lkk (every thread); with suffix, C[0, m) = suffix sums of WB.
// rec: optional trace record (the ends of the two chains)
__device__ __noinline__ double hub_chains(const double* W, const double* WB, double* C, int m, bool suffix,
                                          double* smem, unsigned long long* rec) {
  constexpr int CH = kChainChunk;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = (m + CH - 1) / CH;
  double* LA = smem;           // lkk input, 2 x CH
  double* SB = smem + 2 * CH;  // suffix input, 2 x CH
  double* SO = smem + 4 * CH;  // suffix output, 2 x CH
  double* res = smem + 6 * CH;
  long long busy = 0, waitc = 0;  // trace: chain-thread cycles in the chain / at the group barrier
  if (warp == 0 || warp == 2 || warp == 3) {
    const int gt = warp == 0 ? -1 : (warp - 2) * 32 + lane;  // stager 0..63
    if (gt >= 0) stage_in<8>(LA, W, min(CH, m), gt, 64);
    named_bar(1, 96);
    double s = 0.0;
    for (int c = 0; c < nch; ++c) {
      if (gt >= 0) {
        if (c + 1 < nch) stage_in<8>(LA + ((c + 1) & 1) * CH, W + (c + 1) * CH, min(CH, m - (c + 1) * CH), gt, 64);
      } else if (lane == 0) {
        const long long c0 = clock64();
        s = chain_sum(s, LA + (c & 1) * CH, min(CH, m - c * CH));
        busy += clock64() - c0;
      }
      const long long w0 = clock64();
      named_bar(1, 96);
      waitc += clock64() - w0;
    }
    if (tid == 0) {
      res[0] = s;
      reinterpret_cast<unsigned long long*>(res)[1] = globaltimer_ns();
      reinterpret_cast<long long*>(res)[3] = busy;
      reinterpret_cast<long long*>(res)[4] = waitc;
    }
  } else if (suffix) {
    const int gt = warp == 1 ? -1 : (warp - 4) * 32 + lane;  // stager / writer 0..127
    if (gt >= 0) {
      const int lo = max(0, m - CH);
      stage_in(SB, WB + lo, m - lo, gt, 128);
    }
    named_bar(2, 160);
    double s = 0.0;
    for (int c = 0; c < nch; ++c) {
      const int lo = max(0, m - (c + 1) * CH), hi = m - c * CH;
      if (gt >= 0) {
        if (c + 1 < nch) {
          const int lo2 = max(0, m - (c + 2) * CH);
          stage_in(SB + ((c + 1) & 1) * CH, WB + lo2, lo - lo2, gt, 128);
        }
        if (c >= 1) {  // chunk c-1 = [hi, hi + CH)
          const double* o = SO + ((c - 1) & 1) * CH;
          for (int i = gt; i < CH; i += 128) __stcg(C + hi + i, o[i]);
        }
      } else if (lane == 0) {
        const long long c0 = clock64();
        s = chain_suffix(s, c == 0, SB + (c & 1) * CH, SO + (c & 1) * CH, hi - lo);
        busy += clock64() - c0;
      }
      const long long w0 = clock64();
      named_bar(2, 160);
      waitc += clock64() - w0;
    }
    if (gt >= 0) {  // the last chunk: [0, m - (nch - 1) * CH)
      const double* o = SO + ((nch - 1) & 1) * CH;
      for (int i = gt; i < m - (nch - 1) * CH; i += 128) __stcg(C + i, o[i]);
    }
    if (tid == 32) {
      reinterpret_cast<unsigned long long*>(res)[2] = globaltimer_ns();
      reinterpret_cast<long long*>(res)[5] = busy;
      reinterpret_cast<long long*>(res)[6] = waitc;
    }
  }
  __syncthreads();
  const double lkk = res[0];
  if (rec && threadIdx.x == 0) {  // trace: the ends of the two chains
    hub_step(rec, 8)[2] = reinterpret_cast<unsigned long long*>(res)[1];
    hub_step(rec, 8)[3] = (reinterpret_cast<unsigned long long*>(res)[3] << 32) | reinterpret_cast<unsigned long long*>(res)[4];
    if (suffix) {
      hub_step(rec, 9)[2] = reinterpret_cast<unsigned long long*>(res)[2];
      hub_step(rec, 9)[3] = (reinterpret_cast<unsigned long long*>(res)[5] << 32) | reinterpret_cast<unsigned long long*>(res)[6];
    }
  }
  __syncthreads();  // res / buffers free for the caller
  return lkk;
}

__device__ volatile int g_stop;
// CTA 0 runs the chains; CTAs 1..3 (same SM: 1 CTA per SM is not guaranteed,
// so the launch uses 4 CTAs with smem sized to fit one SM) make noise:
// mode 1 polling (relaxed loads + nanosleep), 2 FP64 chains, 3 shared-memory traffic
__global__ void k(const double* W, const double* WB, double* C, int m, int suffix, unsigned long long* rec, int noise) {
  extern __shared__ double smem[];
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) { hub_step(rec, 8)[0] = globaltimer_ns(); }
    __syncthreads();
    double lkk = hub_chains(W, WB, C, m, suffix, smem, rec);
    if (threadIdx.x == 0) { rec[0] = (unsigned long long)(lkk * 0); g_stop = 1; }
    return;
  }
  unsigned smid, smid0;
  asm("mov.u32 %0, %%smid;" : "=r"(smid));
  double acc = threadIdx.x;
  int it = 0;
  while (!g_stop && ++it < 2000000) {
    if (noise == 1) { acc += W[threadIdx.x & 63]; __nanosleep(256); }
    else if (noise == 2) { for (int q = 0; q < 16; ++q) acc = __dadd_rn(acc, 1e-9 * q); }
    else if (noise == 3) { smem[threadIdx.x] = acc; acc += smem[(threadIdx.x * 7) & 255]; }
    else break;
  }
  (void)smid; (void)smid0;
  if (acc == 12345.678) C[0] = acc;
}
int main() {
  const int m = 2317;
  double *W, *WB, *C; unsigned long long* rec;
  cudaMalloc(&W, m * 8); cudaMalloc(&WB, m * 8); cudaMalloc(&C, m * 8); cudaMallocManaged(&rec, 48 * 8);
  {  // realistic positive weights (zeros: see the value sweep below)
    double* h = new double[m];
    for (int i = 0; i < m; ++i) h[i] = 0.5 + (i * 2654435761u % 1000) * 1e-3;
    cudaMemcpy(W, h, m * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(WB, h, m * 8, cudaMemcpyHostToDevice);
    delete[] h;
  }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40960);
  const int noises[4] = {0, 1, 2, 3};
  for (int ni = 0; ni < 4; ++ni)
  for (int s = 1; s < 2; ++s) for (int rep = 0; rep < 3; ++rep) {
    int zero = 0;
    cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
    // 148 * 4 CTAs of 40 KB: every SM holds 4, CTA 0 shares its SM with 3 noise CTAs
    k<<<noises[ni] ? 148 * 4 : 1, 256, 40960>>>(W, WB, C, m, s, rec, noises[ni]);
    cudaDeviceSynchronize();
    const unsigned long long t0 = hub_step(rec, 8)[0];
    if (rep == 2)
      printf("noise=%d suffix=%d m=%d: lkk %.2f cycles/element (barrier wait %.0f), suffix %.2f cycles/element (barrier wait %.0f)\n", noises[ni], s, m,
             (hub_step(rec, 8)[3] >> 32) / double(m), double(hub_step(rec, 8)[3] & 0xffffffffu),
             s ? (hub_step(rec, 9)[3] >> 32) / double(m) : 0.0, s ? double(hub_step(rec, 9)[3] & 0xffffffffu) : 0.0);
    (void)t0;
  }
  return 0;
}
