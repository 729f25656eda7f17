// C ABI of the device path (include/parac_gpu.h): context, buffers, factor
// driver, downloads. Host orchestration only; all arithmetic is in the
// kernels. There is no CPU fallback: every entry point fails loudly when no
// CUDA device is usable.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/parac_gpu.h"
#include "../host/errors.hpp"
#include "../host/nvtx.hpp"
#include "../host/host_rng.hpp"
#include "factor_kernels.cuh"
#include "solve_kernels.cuh"

namespace parac_gpu {

namespace {
std::atomic<long long> g_launches{0};
}
void note_launches(long long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

namespace {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Failure{internal_error, std::string(what) + ": " + cudaGetErrorString(e)};
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  std::size_t cap = 0;
  void ensure(std::size_t count) {
    if (count <= cap && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const std::size_t c = std::max<std::size_t>(count, 1);
    check(cudaMalloc(&p, c * sizeof(T)), "cudaMalloc");
    cap = c;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Host <-> device copies for caller buffers of any kind. Pinned (page-locked
// or registered) buffers go straight to cudaMemcpyAsync. Pageable buffers --
// the reference's std::vectors in the drop-in path -- would make the driver
// stage them through its own small bounce buffer at ~11-16 GB/s (measured on
// the B200 host); instead they are streamed through two context-owned pinned
// chunks: the DMA of one chunk overlaps the multi-threaded host memcpy of the
// other (~50 GB/s PCIe).
bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// A small persistent pool for the host memcpys of the staged copies (spawning
// threads per chunk cost more than the copies at ~50 GB/s).
class CopyPool {
 public:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const char* e = std::getenv("PARAC_STAGE_THREADS");  // tuning
    nt_ = e ? std::max(1, std::atoi(e)) : static_cast<int>(std::min(8u, hw));
    for (int i = 1; i < nt_; ++i) th_.emplace_back([this, i] { worker(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> l(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void memcpy(void* dst, const void* src, std::size_t bytes) {
    if (nt_ <= 1 || bytes < (std::size_t{4} << 20)) {
      std::memcpy(dst, src, bytes);
      return;
    }
    {
      std::lock_guard<std::mutex> l(m_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      pending_ = nt_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    part(0);
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [this] { return pending_ == 0; });
  }

 private:
  void part(int i) {
    const std::size_t a = (bytes_ * static_cast<std::size_t>(i) / nt_) & ~std::size_t{63};
    const std::size_t b = i + 1 == nt_ ? bytes_ : (bytes_ * static_cast<std::size_t>(i + 1) / nt_) & ~std::size_t{63};
    std::memcpy(dst_ + a, src_ + a, b - a);
  }
  void worker(int i) {
    unsigned long long seen = 0;
    while (true) {
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      part(i);
      std::lock_guard<std::mutex> l(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int nt_ = 1;
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  bool stop_ = false;
  unsigned long long gen_ = 0;
  int pending_ = 0;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  std::size_t bytes_ = 0;
};

struct Stager {
  const std::size_t kChunk = [] {
    const char* e = std::getenv("PARAC_STAGE_CHUNK_MB");  // tuning
    return static_cast<std::size_t>(e ? std::max(1, std::atoi(e)) : 8) << 20;
  }();
  static constexpr std::size_t kDirect = std::size_t{1} << 20;  // smaller copies: plain cudaMemcpyAsync
  char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool armed[2] = {false, false};  // an H2D from buf[i] may still be in flight (ev[i] recorded after it)
  std::unique_ptr<CopyPool> pool;

  void parallel_memcpy(void* dst, const void* src, std::size_t bytes) { pool->memcpy(dst, src, bytes); }
  void ensure() {
    if (buf[0]) return;
    pool = std::make_unique<CopyPool>();
    for (int i = 0; i < 2; ++i) {
      check(cudaMallocHost(&buf[i], kChunk), "cudaMallocHost (staging)");
      check(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "event");
    }
  }
  void release() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventSynchronize(ev[i]);
      if (buf[i]) cudaFreeHost(buf[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
      buf[i] = nullptr;
      ev[i] = nullptr;
      armed[i] = false;
    }
    pool.reset();
  }
  // Enqueues the copy on s. Pageable sources are consumed before return.
  void h2d(void* dst, const void* src, std::size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    if (bytes < kDirect || host_pinned(src)) {
      check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "h2d");
      return;
    }
    ensure();
    int b = 0;
    for (std::size_t off = 0; off < bytes; off += kChunk, b ^= 1) {
      const std::size_t len = std::min(kChunk, bytes - off);
      if (armed[b]) check(cudaEventSynchronize(ev[b]), "staging wait");
      parallel_memcpy(buf[b], static_cast<const char*>(src) + off, len);
      check(cudaMemcpyAsync(static_cast<char*>(dst) + off, buf[b], len, cudaMemcpyHostToDevice, s), "h2d");
      check(cudaEventRecord(ev[b], s), "event");
      armed[b] = true;
    }
  }
  // Synchronous: dst holds the data on return.
  void d2h(void* dst, const void* src, std::size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    if (bytes < kDirect || host_pinned(dst)) {
      check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), "d2h");
      check(cudaStreamSynchronize(s), "d2h sync");
      return;
    }
    ensure();
    const std::size_t nch = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](std::size_t c) {
      const int b = static_cast<int>(c & 1);
      const std::size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      if (armed[b]) check(cudaEventSynchronize(ev[b]), "staging wait");
      check(cudaMemcpyAsync(buf[b], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, s), "d2h");
      check(cudaEventRecord(ev[b], s), "event");
      armed[b] = true;
    };
    issue(0);
    for (std::size_t c = 0; c < nch; ++c) {
      const int b = static_cast<int>(c & 1);
      check(cudaEventSynchronize(ev[b]), "d2h wait");
      armed[b] = false;
      if (c + 1 < nch) issue(c + 1);  // the next chunk's DMA overlaps this chunk's host copy
      const std::size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      parallel_memcpy(static_cast<char*>(dst) + off, buf[b], len);
    }
  }
};

struct Timer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double ms() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
};

}  // namespace
}  // namespace parac_gpu

using namespace parac_gpu;

namespace {
struct Budgets {
  long long ovf, arena, large;
  int c0;
};
}  // namespace

struct parac_gpu_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[6] = {};
  // staged input (label space)
  int n = -1;
  long long nnz = 0;
  long long max_degree = 0;  // of the staged graph (sizes the wide-column slab pool)
  bool needs_hubs = false;   // a run on the staged graph met a column wider than kBigCap
  DevBuf<long long> ptr, scalar;
  DevBuf<int> adj;
  DevBuf<double> w;
  DevBuf<int> perm;
  // factor working state
  DevBuf<int> inv, fdeg, queue, bqueue, samples, col_len, arena_rows, level;
  DevBuf<unsigned long long> cnt;  // dp (low 32) | fills received (high 32)
  DevBuf<int> heavy_list, heavy_count, heavy_key;
  DevBuf<double> heavy_val;
  DevBuf<long long> fwd_ptr, col_start, tiles;
  DevBuf<int> fwd_to;
  DevBuf<double> fwd_w, diag, arena_vals;
  DevBuf<int4> pool0, ovf;
  DevBuf<unsigned> dir;
  DevBuf<char> large_pool;
  DevBuf<HubJob> hub_jobs;  // one per CTA of the elimination grid
  DevBuf<unsigned long long> hub_trace;  // record_times: per hub column phase times
  DevBuf<Ctrl> ctrl;
  DevBuf<unsigned long long> vtimes, vsub;
  bool has_times = false;
  DevBuf<long long> trace_dp;  // on_phase snapshots [3n]
  DevBuf<int> trace_taken;     // [3]
  int trace_n = -1;            // n of the last traced run, -1 none
  Ctrl last_ctrl{};
  long long last_z = 0;
  // resident factor (CSC, position space)
  DevBuf<long long> col_ptr;
  DevBuf<int> rows;
  DevBuf<double> vals;
  int f_n = -1;
  long long f_nnz = 0;
  bool f_has_stats = false;
  bool f_external = false;  // uploaded via parac_gpu_upload_factor
  DevBuf<double> f_diag_ext;
  DevBuf<int> f_perm_ext;
  // batch staging (parac_gpu_upload_batch): problem of each position, first
  // position per problem (count+1), derived sample seed per problem
  int batch_count = 0;
  std::vector<long long> batch_base_h;
  DevBuf<int> pos_pid;
  DevBuf<long long> pid_base, pid_ebase;
  DevBuf<unsigned long long> pid_seed;
  // solve state
  SolveState solve;
  // pinned bounce buffers for pageable caller memory
  Stager stage;
  // streamed assembly (stream_assemble.cu): per-block eliminated counts,
  // chained prefix, claim/publish counters, the streamer's stream, a copy
  // stream for the download, and the mapped pinned progress word
  bool streaming = false;  // the pending attempt assembles beside K3
  DevBuf<int> blk_done, stream_ctl;
  DevBuf<unsigned long long> blk_incl;
  cudaStream_t s_stream = nullptr, s_copy = nullptr;
  unsigned long long* blkh_h = nullptr;  // [blkh_cap] per-block release words (host view)
  unsigned long long* blkh_d = nullptr;  // (device view)
  std::size_t blkh_cap = 0;
  // batch: streamer blocks that never straddle problems (positions, nb+1),
  // each block's member and that member's first block, the claim order
  // (members interleaved), and the member regions of a streamed batch
  // (stream_assemble.cu): member p's entries at region[p], its local col_ptr
  // in lcol[base_p + p ...]
  std::vector<int> blk_k0_h, blk_mem_h, blk_first_h, claim_h;
  std::vector<long long> batch_ebase_h;
  DevBuf<int> blk_k0, blk_first, claim, overflow;
  DevBuf<long long> region, reg_cap, lcol;
  bool batch_regions = false;                 // the resident batch factor is in the region layout
  std::vector<long long> region_h, reg_cap_h, batch_z_h;  // per member: region start, capacity, off-diagonal count
  // a factorization launched by parac_gpu_factor_begin, completed by _end
  bool pending = false;
  std::uint64_t p_seed = 0;
  parac_gpu_options p_opt{};
  Budgets p_b{};
  int p_attempts = 0;
  double p_failed_ms = 0.0;
  std::chrono::steady_clock::time_point p_t0;
};

namespace {

void activate(parac_gpu_ctx* ctx) { check(cudaSetDevice(ctx->device), "cudaSetDevice"); }

int device_sms(parac_gpu_ctx* ctx) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  return sms;
}

void require_ctx_any(parac_gpu_ctx* ctx) {
  if (!ctx) throw Failure{internal_error, "null context"};
  activate(ctx);
}
// Every entry point but parac_gpu_factor_end: the buffers of a pending
// factorization (parac_gpu_factor_begin) are in use on the device.
void require_ctx(parac_gpu_ctx* ctx) {
  require_ctx_any(ctx);
  if (ctx->pending) throw Failure{internal_error, "a factorization is pending (call parac_gpu_factor_end)"};
}

Budgets default_budgets(int n, long long E, long long max_degree, const parac_gpu_options& o,
                        std::size_t own_pool_bytes = 0) {
  Budgets b;
  const long long base = E + n;
  // 64 preallocated slots per position cover the fill count of ~99.5% of
  // 128^3 positions (p99 66), so the directory lookup is rare.
  // Preallocated fill slots per position: as many as 40% of the device's
  // free memory allows (the context's own fill pool counted as free, so the
  // choice is stable across calls; at least ~17.6 GB's worth), up to 512, at
  // least 64. The widest (latest, critical-path) columns gather
  // hundreds of fills; beyond the preallocated slots each costs directory
  // round trips on the emission and gather paths. Measured K3 at 128^3 by
  // slots: 32: 20.7, 64: 20.55, 128: 20.3, 256: 19.91, 384: 19.60, 512: 19.49,
  // 1024: 19.51 ms; 27-point 96^3 256 -> 512: 30.31 -> 29.43 ms. A compact
  // store (fewer slots, more overflow) is slower, not faster.
  if (o.first_chunk > 0) {
    b.c0 = o.first_chunk;
  } else {
    std::size_t free_b = 0, total_b = 0;
    long long budget = 17600000000LL;  // (measured: the 64 x 64^3 batch, 64 -> 256 slots: K3 64.1 -> 62.5 ms)
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess)
      budget = std::max(budget, static_cast<long long>(0.4 * static_cast<double>(free_b + own_pool_bytes)));
    const long long cap = budget / (16LL * std::max(n, 1));
    b.c0 = cap >= 512 ? 512 : cap >= 256 ? 256 : cap >= 128 ? 128 : 64;
  }
  // hub graphs: fills concentrate on a few positions whose overflow chunks
  // grow geometrically (up to 2x waste), and raw columns are wide
  const bool hubs = max_degree > 512;
  b.ovf = o.fill_pool_entries >= 0 ? o.fill_pool_entries : (hubs ? 8 : 4) * base + 4096;
  b.arena = o.column_arena_entries >= 0 ? o.column_arena_entries : (hubs ? 8 : 6) * base + 4096;
  // wide-column slabs (R > 1024): each big CTA's slab grows geometrically to
  // the widest raw column it meets; hub graphs (R-MAT: raw columns up to ~10^6
  // entries with fills) need ~4x the graph size, which the first attempt
  // should get instead of failing after seconds and retrying
  b.large = (hubs ? 4 : 1) * base + 65536;
  return b;
}

// Streamed assembly beside K3 (stream_assemble.cu): on by default
// (PARAC_STREAM=0: assemble after K3), PARAC_STREAM_CTAS CTAs
int stream_ctas(const parac_gpu_ctx* ctx) {
  const char* e = std::getenv("PARAC_STREAM_CTAS");
  // batches: 16 (64 x 64^3: 8 CTAs fell behind the elimination by 10 ms; 16
  // and 32 kept up, 16 with the shorter K3)
  return e ? std::max(1, std::min(64, std::atoi(e))) : ctx->batch_count > 0 ? 16 : 8;
}
bool stream_wanted(const parac_gpu_ctx* ctx) {
  const char* e = std::getenv("PARAC_STREAM");
  const int m = e ? std::atoi(e) : 1;
  // PARAC_STREAM_BATCH=0: batches assemble after K3 (their streamed layout is
  // per member, stream_assemble.cu; 64 x 64^3 e2e 148.5 -> 114.6 ms, device
  // time unchanged)
  const char* eb = std::getenv("PARAC_STREAM_BATCH");
  if (ctx->batch_count > 0 && eb && std::atoi(eb) == 0) return false;
  return (m == 1 || m == 3) && ctx->n > 0;
}
// PARAC_STREAM=3 (diagnostics): the streamer runs after K3 on K3's stream --
// its throughput alone
bool stream_serial() {
  const char* e = std::getenv("PARAC_STREAM");
  return e && std::atoi(e) == 3;
}
// PARAC_STREAM=2 (diagnostics): K3 counts the blocks' columns, the assembly
// still runs after it -- the cost of the counting alone
bool stream_count_only() {
  const char* e = std::getenv("PARAC_STREAM");
  return e && std::atoi(e) == 2;
}
void ensure_stream_resources(parac_gpu_ctx* ctx) {
  if (!ctx->s_stream) check(cudaStreamCreateWithFlags(&ctx->s_stream, cudaStreamNonBlocking), "stream");
  if (!ctx->s_copy) check(cudaStreamCreateWithFlags(&ctx->s_copy, cudaStreamNonBlocking), "stream");
}

// The streamer's per-block release words (mapped pinned), nblk of them.
void ensure_release_words(parac_gpu_ctx* ctx, std::size_t nblk) {
  if (nblk <= ctx->blkh_cap) return;
  if (ctx->blkh_h) cudaFreeHost(ctx->blkh_h);
  ctx->blkh_h = nullptr;
  ctx->blkh_cap = 0;
  void* h = nullptr;
  check(cudaHostAlloc(&h, sizeof(unsigned long long) * nblk, cudaHostAllocMapped), "cudaHostAlloc (release words)");
  ctx->blkh_h = static_cast<unsigned long long*>(h);
  void* dp = nullptr;
  check(cudaHostGetDevicePointer(&dp, h, 0), "cudaHostGetDevicePointer");
  ctx->blkh_d = static_cast<unsigned long long*>(dp);
  ctx->blkh_cap = nblk;
}

// Launch half of one attempt of the factorization with the given budgets
// (stream-ordered; complete_factor waits for it).
void launch_factor(parac_gpu_ctx* ctx, std::uint64_t seed, const parac_gpu_options& o,
                   const Budgets& b) {
  const int n = ctx->n;
  const long long E = ctx->nnz / 2;
  cudaStream_t s = ctx->stream;
  const std::size_t nn = static_cast<std::size_t>(std::max(n, 1));
  ctx->inv.ensure(nn);
  ctx->fdeg.ensure(nn);
  ctx->cnt.ensure(nn);
  ctx->queue.ensure(nn);
  ctx->bqueue.ensure(nn);
  ctx->samples.ensure(nn);
  ctx->level.ensure(nn);
  ctx->col_len.ensure(nn);
  ctx->col_start.ensure(nn);
  ctx->diag.ensure(nn);
  ctx->fwd_ptr.ensure(nn + 1);
  ctx->fwd_to.ensure(static_cast<std::size_t>(std::max<long long>(E, 1)));
  ctx->fwd_w.ensure(static_cast<std::size_t>(std::max<long long>(E, 1)));
  ctx->heavy_list.ensure(nn);
  ctx->heavy_count.ensure(1);
  ctx->heavy_key.ensure(static_cast<std::size_t>(std::max<long long>(E, 1)));
  ctx->heavy_val.ensure(static_cast<std::size_t>(std::max<long long>(E, 1)));
  ctx->pool0.ensure(nn * static_cast<std::size_t>(b.c0));
  ctx->dir.ensure(nn * kDirChunks);
  ctx->ovf.ensure(static_cast<std::size_t>(std::max<long long>(b.ovf, 1)));
  ctx->arena_rows.ensure(static_cast<std::size_t>(std::max<long long>(b.arena, 1)));
  ctx->arena_vals.ensure(static_cast<std::size_t>(std::max<long long>(b.arena, 1)));
  ctx->large_pool.ensure(static_cast<std::size_t>(std::max<long long>(b.large, 1)) * kSlabEntryBytes);
  const int hub_jobs = eliminate_occupancy_grid(ctx->device);
  ctx->hub_jobs.ensure(static_cast<std::size_t>(hub_jobs));
  ctx->rows.ensure(static_cast<std::size_t>(std::max<long long>(b.arena, 1)));
  ctx->vals.ensure(static_cast<std::size_t>(std::max<long long>(b.arena, 1)));
  ctx->ctrl.ensure(1);
  ctx->tiles.ensure(static_cast<std::size_t>(std::max<long long>(scan_tiles(n) + 1, initial_ready_scratch(n))));
  ctx->col_ptr.ensure(nn + 1);

  FactorDev d{};
  d.n = n;
  d.ptr = ctx->ptr.p;
  d.adj = ctx->adj.p;
  d.w = ctx->w.p;
  d.perm = ctx->perm.p;
  d.inv = ctx->inv.p;
  d.fwd_ptr = ctx->fwd_ptr.p;
  d.fwd_to = ctx->fwd_to.p;
  d.fwd_w = ctx->fwd_w.p;
  d.fdeg = ctx->fdeg.p;
  d.heavy_list = ctx->heavy_list.p;
  d.heavy_count = ctx->heavy_count.p;
  d.heavy_key = ctx->heavy_key.p;
  d.heavy_val = ctx->heavy_val.p;
  d.cnt = ctx->cnt.p;
  d.queue = ctx->queue.p;
  d.bqueue = ctx->bqueue.p;
  d.pool0 = ctx->pool0.p;
  d.dir = ctx->dir.p;
  d.ovf = ctx->ovf.p;
  d.ovf_cap = b.ovf;
  d.c0 = b.c0;
  d.col_start = ctx->col_start.p;
  d.col_len = ctx->col_len.p;
  d.diag = ctx->diag.p;
  d.arena_rows = ctx->arena_rows.p;
  d.arena_vals = ctx->arena_vals.p;
  d.arena_cap = b.arena;
  d.samples = ctx->samples.p;
  d.level = ctx->level.p;
  d.large_pool = ctx->large_pool.p;
  d.hub_jobs = ctx->hub_jobs.p;
  {  // PARAC_HUB_LINGER_NS: how long a helper stays with a hub job between its phases (tuning)
    const char* e = std::getenv("PARAC_HUB_LINGER_NS");
    d.hub_linger_ns = e ? std::strtoull(e, nullptr, 10) : 40000ull;
    const char* hp = std::getenv("PARAC_HUB_PIPE");
    d.hub_pipe = hp ? std::atoi(hp) : 1;
    const char* w = std::getenv("PARAC_HUB_WAIT_NS");
    d.hub_wait_ns = w ? static_cast<unsigned>(std::atoi(w)) : 4096u;
    // the kernel instance with the hub path on graphs with hub vertices, or
    // once a run on this graph met a column wider than kBigCap (PARAC_HUBS=0/1
    // overrides the first choice; tuning / tests)
    const char* hh = std::getenv("PARAC_HUBS");
    d.hubs = ctx->needs_hubs || (hh ? std::atoi(hh) != 0 : ctx->max_degree > 512);
  }
  d.large_cap = b.large;
  d.ctrl = ctx->ctrl.p;
  d.sample_seed = derive_seed(seed, kSaltSampling);
  d.pos_pid = ctx->batch_count > 0 ? ctx->pos_pid.p : nullptr;
  d.pid_base = ctx->batch_count > 0 ? ctx->pid_base.p : nullptr;
  d.pid_seed = ctx->batch_count > 0 ? ctx->pid_seed.p : nullptr;
  const double wd = o.watchdog_seconds > 0 ? o.watchdog_seconds : 60.0;
  d.watchdog_ns = static_cast<unsigned long long>(wd * 1e9);
  d.verify = o.verify;
  {  // PARAC_CLAIM_SLEEP="a,b,c" (ns) overrides the claim backoff tiers (tuning)
    unsigned t[3] = {128, 1024, 4096};  // measured: 2D 256^2 1.77 -> 1.40 ms, 128^3 -1% vs 512,4096,16384
    if (const char* e = std::getenv("PARAC_CLAIM_SLEEP")) std::sscanf(e, "%u,%u,%u", &t[0], &t[1], &t[2]);
    for (int i = 0; i < 3; ++i) d.sleep_ns[i] = t[i];
    const char* kp = std::getenv("PARAC_KEEP");
    d.keep_pos = kp && std::string(kp) == "width" ? 0 : 1;  // default: lowest position
    const char* kl = std::getenv("PARAC_KEEP_LIMIT");
    d.keep_limit = kl ? std::max(1, std::atoi(kl)) : 1 << 30;
    const char* bl = std::getenv("PARAC_BIG_LAYOUT");
    d.big_layout = bl ? std::atoi(bl) : 1;  // measured: 128^3 -2.3%, 27-point -2.9%, 2D -2.3% vs 0
    // routing threshold: 64 on sparse graphs (mean degree <= 8), 128 on denser
    // ones (see kSmallCap); PARAC_SMALL_CAP overrides (tuning)
    const double mean_deg = n > 0 ? 2.0 * static_cast<double>(E) / n : 0.0;
    d.small_cap = mean_deg <= 8.0 ? 64 : 96;
    if (const char* sc = std::getenv("PARAC_SMALL_CAP")) d.small_cap = std::atoi(sc);
    d.small_cap = std::max(1, std::min(d.small_cap, kSmallCap));
    const char* df = std::getenv("PARAC_DISCARD_FILLS");
    // only when every position's slot block is whole 128-byte lines (lines
    // are never shared between positions). Off by default: measured 128^3
    // K3 DRAM traffic 2.00 -> 1.81 GB but +0.8% time (the discards' issue
    // cost outweighs the saved write-backs on this latency-bound kernel)
    d.discard_fills = (df ? std::atoi(df) : 0) && b.c0 % 8 == 0;
  }
  d.delay_ns = o.delay_ns;
  d.vtimes = nullptr;
  d.vsub = nullptr;
  d.hub_trace = nullptr;
  d.trace_k = -1;
  d.trace_dp = nullptr;
  d.trace_taken = nullptr;
  ctx->trace_n = -1;
  if (o.trace_phases) {
    if (o.trace_position < 0 || o.trace_position >= n)
      throw Failure{dimension_mismatch, "trace_position outside [0, n)"};
    ctx->trace_dp.ensure(3 * nn);
    ctx->trace_taken.ensure(3);
    check(cudaMemsetAsync(ctx->trace_dp.p, 0xff, 3 * nn * sizeof(long long), s), "memset");
    check(cudaMemsetAsync(ctx->trace_taken.p, 0, 3 * sizeof(int), s), "memset");
    d.trace_k = o.trace_position;
    d.trace_dp = ctx->trace_dp.p;
    d.trace_taken = ctx->trace_taken.p;
    ctx->trace_n = n;
  }
  ctx->has_times = o.record_times != 0;
  if (o.record_times) {
    ctx->vtimes.ensure(8 * nn);
    check(cudaMemsetAsync(ctx->vtimes.p, 0, 8 * nn * sizeof(unsigned long long), s), "memset");
    d.vtimes = ctx->vtimes.p;
    ctx->vsub.ensure(12 * nn);  // 8 sub-phase stamps + 4 cycle counters (rank-sort diagnostics)
    check(cudaMemsetAsync(ctx->vsub.p, 0, 12 * nn * sizeof(unsigned long long), s), "memset");
    d.vsub = ctx->vsub.p;
    ctx->hub_trace.ensure(static_cast<std::size_t>(kHubTraceCap) * kHubTraceWords);
    check(cudaMemsetAsync(ctx->hub_trace.p, 0, sizeof(unsigned long long) * kHubTraceCap * kHubTraceWords, s),
          "memset");
    d.hub_trace = ctx->hub_trace.p;
  }

  d.blk_done = nullptr;
  const bool count = ctx->streaming || stream_count_only();
  if (count) {
    ensure_stream_resources(ctx);
    const std::size_t nb = static_cast<std::size_t>((n + kStreamBlock - 1) >> kStreamShift);
    const std::size_t nblk = ctx->batch_count > 0 ? ctx->blk_k0_h.size() - 1 : nb;
    ctx->blk_done.ensure(nb);
    ctx->blk_incl.ensure(std::max<std::size_t>(nblk, 1));
    ctx->stream_ctl.ensure(2);
    ensure_release_words(ctx, std::max<std::size_t>(nblk, 1));
    // no stream work of an earlier attempt is in flight
    std::memset(ctx->blkh_h, 0, sizeof(unsigned long long) * std::max<std::size_t>(nblk, 1));
    d.blk_done = ctx->blk_done.p;
  }
  if (ctx->streaming && ctx->batch_count > 0) {  // member regions: a share of the column arena's budget each, by size
    const int count = ctx->batch_count;
    const std::vector<long long>& base = ctx->batch_base_h;
    const std::vector<long long>& eb = ctx->batch_ebase_h;
    const double tot_w = static_cast<double>(std::max<long long>(E + n, 1));
    ctx->region_h.assign(count + 1, 0);
    std::vector<long long>& cap = ctx->reg_cap_h;
    cap.assign(count, 0);
    for (int i = 0; i < count; ++i) {
      const long long w = (eb[i + 1] - eb[i]) / 2 + (base[i + 1] - base[i]);
      cap[i] = static_cast<long long>(static_cast<double>(b.arena) * (static_cast<double>(w) / tot_w)) + 4096;
      ctx->region_h[i + 1] = ctx->region_h[i] + cap[i];
    }
    const std::size_t rtot = static_cast<std::size_t>(std::max<long long>(ctx->region_h[count], 1));
    ctx->rows.ensure(rtot);
    ctx->vals.ensure(rtot);
    ctx->region.ensure(count);
    ctx->reg_cap.ensure(count);
    ctx->lcol.ensure(static_cast<std::size_t>(n) + count);
    ctx->overflow.ensure(1);
    check(cudaMemcpyAsync(ctx->region.p, ctx->region_h.data(), sizeof(long long) * count, cudaMemcpyHostToDevice, s),
          "h2d");
    check(cudaMemcpyAsync(ctx->reg_cap.p, cap.data(), sizeof(long long) * count, cudaMemcpyHostToDevice, s), "h2d");
    check(cudaMemsetAsync(ctx->overflow.p, 0, sizeof(int), s), "memset");
  }
  check(cudaEventRecord(ctx->ev[0], s), "event");
  if (count) {
    const std::size_t nb = static_cast<std::size_t>((n + kStreamBlock - 1) >> kStreamShift);
    check(cudaMemsetAsync(ctx->blk_done.p, 0, nb * sizeof(int), s), "memset");
    const std::size_t nblk = ctx->batch_count > 0 ? ctx->blk_k0_h.size() - 1 : nb;
    check(cudaMemsetAsync(ctx->blk_incl.p, 0, std::max<std::size_t>(nblk, 1) * sizeof(unsigned long long), s), "memset");
    check(cudaMemsetAsync(ctx->stream_ctl.p, 0, 2 * sizeof(int), s), "memset");
  }
  check(cudaMemsetAsync(ctx->inv.p, 0xff, nn * sizeof(int), s), "memset");
  check(cudaMemsetAsync(ctx->dir.p, 0, nn * kDirChunks * sizeof(unsigned), s), "memset");
  check(cudaMemsetAsync(ctx->ctrl.p, 0, sizeof(Ctrl), s), "memset");
  check(cudaMemsetAsync(ctx->hub_jobs.p, 0, static_cast<std::size_t>(hub_jobs) * sizeof(HubJob), s), "memset");
  check(launch_pos_graph(d, ctx->tiles.p, s), "pos_graph launch");
  check(launch_initial_ready(d, ctx->tiles.p, s), "initial_ready launch");
  check(cudaEventRecord(ctx->ev[1], s), "event");
  int grid = 0;
  const int sctas = ctx->streaming ? stream_ctas(ctx) : 0;
  const bool serial = ctx->streaming && stream_serial();
  check(launch_eliminate(d, o.grid_ctas, serial ? 0 : sctas, s, &grid), "eliminate launch");
  if (serial) check(cudaEventRecord(ctx->ev[2], s), "event");
  if (ctx->streaming) {  // the assembly beside K3, on its own stream (after K1/K2)
    StreamDev sd{};
    sd.n = n;
    const bool batch = ctx->batch_count > 0;
    sd.nb = batch ? static_cast<int>(ctx->blk_k0_h.size()) - 1 : (n + kStreamBlock - 1) >> kStreamShift;
    sd.blk_k0 = batch ? ctx->blk_k0.p : nullptr;
    sd.pos_pid = batch ? ctx->pos_pid.p : nullptr;
    sd.pid_base = batch ? ctx->pid_base.p : nullptr;
    if (batch) {
      sd.claim = ctx->claim.p;
      sd.blk_first = ctx->blk_first.p;
      sd.region = ctx->region.p;
      sd.reg_cap = ctx->reg_cap.p;
      sd.lcol = ctx->lcol.p;
      sd.overflow = ctx->overflow.p;
    }
    sd.blk_done = ctx->blk_done.p;
    sd.col_len = ctx->col_len.p;
    sd.col_start = ctx->col_start.p;
    sd.arena_rows = ctx->arena_rows.p;
    sd.arena_vals = ctx->arena_vals.p;
    sd.col_ptr = ctx->col_ptr.p;
    sd.rows = ctx->rows.p;
    sd.vals = ctx->vals.p;
    sd.blk_incl = ctx->blk_incl.p;
    sd.next_blk = ctx->stream_ctl.p;
    sd.host_blk = ctx->blkh_d;
    sd.ctrl = ctx->ctrl.p;
    {  // PARAC_STREAM_START=f: the streamer starts once f*n positions are eliminated
      const char* e = std::getenv("PARAC_STREAM_START");
      const double f = e ? std::atof(e) : 0.0;
      sd.start_after = serial ? 0 : static_cast<int>(f * n);
    }
    cudaStream_t ss = serial ? s : ctx->s_stream;
    if (!serial) check(cudaStreamWaitEvent(ss, ctx->ev[1], 0), "stream wait");
    check(launch_stream_assemble(sd, sctas, ss), "stream assemble launch");
    check(cudaEventRecord(ctx->ev[4], ss), "event");
  }
  if (!serial) check(cudaEventRecord(ctx->ev[2], s), "event");
  if (ctx->streaming) {
    check(launch_sum_samples(d, s), "sum samples");
    check(cudaStreamWaitEvent(s, ctx->ev[4], 0), "stream join");
  } else {
    check(launch_assemble(d, ctx->col_ptr.p, ctx->rows.p, ctx->vals.p, ctx->tiles.p, s), "assemble");
  }
  check(cudaEventRecord(ctx->ev[3], s), "event");
}

// Where the completion half copies the factor (any pointer may be null;
// rows/values hold cap entries).
struct HostOut {
  std::int64_t* col_ptr;
  std::int32_t* rows;
  double* values;
  double* diag;
  long long cap;
};

// Device -> host copy of [off, off + bytes) of one array: pinned targets by
// DMA on the copy stream (waited for at the end), pageable ones through the
// staging buffers (synchronous)
void copy_range(parac_gpu_ctx* ctx, void* dst, const void* src, std::size_t bytes) {
  if (!dst || bytes == 0) return;
  if (host_pinned(dst)) check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->s_copy), "d2h");
  else ctx->stage.d2h(dst, src, bytes, ctx->s_copy);
}

// The download beside the elimination: polls the streamer's progress word and
// copies each newly final range (entries, and the blocks' col_ptr/diag) while
// K3 runs. Returns once every block is copied or the device work ended
// without it (an aborted attempt; the caller reads the status).
void stream_download(parac_gpu_ctx* ctx, const HostOut& out) {
  const int n = ctx->n;
  const int nb = (n + kStreamBlock - 1) >> kStreamShift;
  volatile unsigned long long* rel = ctx->blkh_h;
  const long long kMinEntries = 1 << 19;  // ~6 MB of rows+values per round of copies
  int done_b = 0, seen_b = 0;
  long long done_z = 0;
  auto take = [&](int) {
    while (seen_b < nb && (rel[seen_b] >> 63)) ++seen_b;  // the contiguous released prefix
    const int pb = seen_b;
    const long long pz = pb > 0 ? static_cast<long long>(rel[pb - 1] & ~(1ull << 63)) : 0;
    if (pb <= done_b || (pb < nb && pz - done_z < kMinEntries)) return;
    const long long p0 = static_cast<long long>(done_b) << kStreamShift;
    const long long p1 = std::min<long long>(static_cast<long long>(pb) << kStreamShift, n);
    const long long z1 = std::min(pz, out.cap);
    if (z1 > done_z) {
      copy_range(ctx, out.rows ? out.rows + done_z : nullptr, ctx->rows.p + done_z, sizeof(int) * (z1 - done_z));
      copy_range(ctx, out.values ? out.values + done_z : nullptr, ctx->vals.p + done_z,
                 sizeof(double) * (z1 - done_z));
    }
    const long long q1 = pb == nb ? p1 + 1 : p1;  // col_ptr[n] with the last block
    copy_range(ctx, out.col_ptr ? out.col_ptr + p0 : nullptr, ctx->col_ptr.p + p0, sizeof(long long) * (q1 - p0));
    copy_range(ctx, out.diag ? out.diag + p0 : nullptr, ctx->diag.p + p0, sizeof(double) * (p1 - p0));
    done_b = pb;
    done_z = pz;
  };
  while (done_b < nb) {
    take(0);
    if (done_b == nb) break;
    if (cudaEventQuery(ctx->ev[3]) == cudaSuccess) {  // device work over: the words are final
      take(0);
      break;
    }
    std::this_thread::yield();
  }
  check(cudaStreamSynchronize(ctx->s_copy), "d2h sync");
}

// Per-problem outputs of a batch (each array: problem i's buffer, or null).
struct BatchOut {
  std::int64_t* const* col_ptr;
  std::int32_t* const* rows;
  double* const* values;
  double* const* diag;
  const std::int64_t* caps;
  bool short_cap = false;  // some problem's factor exceeded its capacity
  bool redo = false;       // a member outgrew its region: downloaded again from the union CSC
};

// The batch download beside the elimination (member regions). Member p's
// blocks release independently of the other members'; for each member the
// contiguous released prefix of its blocks is copied: its local col_ptr
// (lcol), diag, and its entries from its region -- all in its own position and
// entry space, so nothing is rebased on the host.
void stream_download_batch(parac_gpu_ctx* ctx, BatchOut& out) {
  const int count = ctx->batch_count;
  const std::vector<long long>& base = ctx->batch_base_h;
  const std::vector<int>& bk = ctx->blk_k0_h;
  const int nb = static_cast<int>(bk.size()) - 1;
  volatile unsigned long long* rel = ctx->blkh_h;
  constexpr unsigned long long kRel = 1ull << 63;
  std::vector<int> cur(count, -1), last(count, -1);
  for (int b = 0; b < nb; ++b) {
    const int p = ctx->blk_mem_h[b];
    if (cur[p] < 0) cur[p] = b;
    last[p] = b;
  }
  std::vector<long long> dz(count, 0);
  std::vector<int> active;
  for (int p = 0; p < count; ++p)
    if (cur[p] >= 0) active.push_back(p);
  const long long kMinEntries = 1 << 19;
  auto pass = [&](bool final_pass) {
    for (std::size_t ai = 0; ai < active.size();) {
      const int p = active[ai];
      int c = cur[p];
      while (c <= last[p] && (rel[c] & kRel)) ++c;
      const long long z1 = c > cur[p] ? static_cast<long long>(rel[c - 1] & ~kRel) : dz[p];
      const bool done = c > last[p];
      if (c == cur[p] || (!done && !final_pass && z1 - dz[p] < kMinEntries)) {
        ++ai;
        continue;
      }
      const long long P0 = bk[cur[p]], P1 = bk[c];  // positions [P0, P1): col_ptr through P1
      if (out.col_ptr && out.col_ptr[p])
        copy_range(ctx, out.col_ptr[p] + (P0 - base[p]), ctx->lcol.p + P0 + p, sizeof(long long) * (P1 - P0 + 1));
      if (out.diag && out.diag[p])
        copy_range(ctx, out.diag[p] + (P0 - base[p]), ctx->diag.p + P0, sizeof(double) * (P1 - P0));
      const long long cap = out.caps ? out.caps[p] : 0;
      const long long c1 = std::min(z1, cap);
      if (c1 > dz[p]) {
        const long long r0 = ctx->region_h[p];
        if (out.rows && out.rows[p])
          copy_range(ctx, out.rows[p] + dz[p], ctx->rows.p + r0 + dz[p], sizeof(int) * (c1 - dz[p]));
        if (out.values && out.values[p])
          copy_range(ctx, out.values[p] + dz[p], ctx->vals.p + r0 + dz[p], sizeof(double) * (c1 - dz[p]));
      }
      if (z1 > cap) out.short_cap = true;
      dz[p] = z1;
      cur[p] = c;
      if (done) {
        active[ai] = active.back();
        active.pop_back();
      } else {
        ++ai;
      }
    }
  };
  while (!active.empty()) {
    pass(false);
    if (active.empty()) break;
    if (cudaEventQuery(ctx->ev[3]) == cudaSuccess) {
      pass(true);
      break;
    }
    std::this_thread::yield();
  }
  check(cudaStreamSynchronize(ctx->s_copy), "d2h sync");
  for (int p = 0; p < count; ++p)  // members without vertices: col_ptr = {0}
    if (base[p + 1] == base[p] && out.col_ptr && out.col_ptr[p]) out.col_ptr[p][0] = 0;
}

// Completion half: the streamed download (when outputs are given and the
// attempt streams), then the status. Returns status.
int complete_factor(parac_gpu_ctx* ctx, const parac_gpu_options& o, const Budgets& b, const HostOut* out,
                    BatchOut* bout = nullptr) {
  const int n = ctx->n;
  cudaStream_t s = ctx->stream;
  const double wd = o.watchdog_seconds > 0 ? o.watchdog_seconds : 60.0;
  if (out && ctx->streaming) stream_download(ctx, *out);
  if (bout && ctx->streaming) stream_download_batch(ctx, *bout);
  Ctrl c{};
  long long z = 0;
  check(cudaMemcpyAsync(&c, ctx->ctrl.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, s), "ctrl copy");
  check(cudaMemcpyAsync(&z, ctx->col_ptr.p + n, sizeof(long long), cudaMemcpyDeviceToHost, s), "z copy");
  check(cudaStreamSynchronize(s), "factor sync");
  ctx->last_ctrl = c;
  ctx->last_z = z;
  if (c.status == kStatusNeedHubs) {  // re-run with the hub path (parac_gpu_factor_resident)
    ctx->f_n = -1;
    ctx->needs_hubs = true;
    return c.status;
  }
  if (c.status != 0) {
    ctx->f_n = -1;
    std::string msg;
    if (c.status == arena_exhausted)
      msg = "pool budget exhausted at position " + std::to_string(c.err_info) +
            " (overflow used " + std::to_string(c.ovf_bump) + "/" + std::to_string(b.ovf) +
            ", arena " + std::to_string(c.arena_bump) + "/" + std::to_string(b.arena) +
            ", large " + std::to_string(c.large_bump) + "/" + std::to_string(b.large) + ")";
    else if (c.status == queue_stall)
      msg = "no elimination for " + std::to_string(wd) + "s while waiting on queue slot " +
            std::to_string(c.err_info) + " (" + std::to_string(c.q_tail) + "/" +
            std::to_string(n) + " published)";
    else if (c.status == not_a_permutation)
      msg = "ordering is not a permutation (vertex " + std::to_string(c.err_info) + ")";
    else
      msg = "device verify failure at position " + std::to_string(c.err_info);
    set_last_error(std::string(errc_name(c.status)) + ": " + msg);
    return c.status;
  }
  return 0;
}

}  // namespace

extern "C" {

int parac_gpu_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

int64_t parac_gpu_launch_count(void) { return g_launches.load(); }

void parac_gpu_default_options(parac_gpu_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->fill_pool_entries = -1;
  o->column_arena_entries = -1;
  o->first_chunk = 0;
  o->watchdog_seconds = 60.0;
  o->record_stats = 1;
  o->verify = 0;
  o->grid_ctas = 0;
  o->delay_ns = 0;
}

int parac_gpu_create(int32_t device, parac_gpu_ctx** out) {
  return guarded([&] {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
      throw Failure{internal_error, std::string("no CUDA device available (") +
                                        cudaGetErrorString(e) +
                                        "); this library has no CPU fallback"};
    if (device < 0 || device >= count) throw Failure{internal_error, "device ordinal out of range"};
    auto* ctx = new parac_gpu_ctx;
    ctx->device = device;
    try {
      activate(ctx);
      check(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
      for (auto& ev : ctx->ev) check(cudaEventCreate(&ev), "event");
    } catch (...) {
      delete ctx;
      throw;
    }
    *out = ctx;
  });
}

void parac_gpu_destroy(parac_gpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->ptr.release(); ctx->scalar.release(); ctx->adj.release(); ctx->w.release(); ctx->perm.release();
  ctx->heavy_list.release(); ctx->heavy_count.release(); ctx->heavy_key.release(); ctx->heavy_val.release();
  ctx->inv.release(); ctx->fdeg.release(); ctx->cnt.release(); ctx->level.release(); ctx->queue.release(); ctx->bqueue.release();
  ctx->samples.release(); ctx->col_len.release();
  ctx->arena_rows.release(); ctx->fwd_ptr.release(); ctx->col_start.release();
  ctx->tiles.release(); ctx->fwd_to.release(); ctx->fwd_w.release(); ctx->diag.release();
  ctx->arena_vals.release(); ctx->pool0.release(); ctx->ovf.release(); ctx->dir.release();
  ctx->large_pool.release(); ctx->hub_jobs.release(); ctx->hub_trace.release(); ctx->ctrl.release(); ctx->vtimes.release(); ctx->vsub.release(); ctx->col_ptr.release(); ctx->rows.release();
  ctx->vals.release(); ctx->f_diag_ext.release(); ctx->f_perm_ext.release();
  solve_release(ctx->solve);
  ctx->stage.release();
  if (ctx->s_stream) cudaStreamSynchronize(ctx->s_stream);
  if (ctx->s_copy) cudaStreamSynchronize(ctx->s_copy);
  ctx->blk_done.release(); ctx->stream_ctl.release(); ctx->blk_incl.release();
  if (ctx->blkh_h) cudaFreeHost(ctx->blkh_h);
  ctx->blk_k0.release();
  if (ctx->s_stream) cudaStreamDestroy(ctx->s_stream);
  if (ctx->s_copy) cudaStreamDestroy(ctx->s_copy);
  for (auto& ev : ctx->ev) cudaEventDestroy(ev);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int parac_gpu_ordering_nnz_sort(parac_gpu_ctx* ctx, const parac_csr* g, uint64_t seed, int32_t* perm) {
  NvtxRange nvtx_range("parac_gpu_ordering_nnz_sort");
  return guarded([&] {
    require_ctx(ctx);
    if (!g || g->n < 0 || (g->n > 0 && (!g->ptr || !perm))) throw Failure{dimension_mismatch, "bad graph"};
    const int n = g->n;
    if (n == 0) return;
    cudaStream_t s = ctx->stream;
    long long* d_ptr = nullptr;
    int* d_perm = nullptr;
    check(cudaMallocAsync(&d_ptr, sizeof(long long) * (static_cast<std::size_t>(n) + 1), s), "alloc");
    check(cudaMallocAsync(&d_perm, sizeof(int) * static_cast<std::size_t>(n), s), "alloc");
    check(cudaMemcpyAsync(d_ptr, g->ptr, sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, s), "h2d");
    nnz_sort_device(n, d_ptr, derive_seed(seed, kSaltTieBreak), d_perm, s, device_sms(ctx));
    check(cudaMemcpyAsync(perm, d_perm, sizeof(int) * n, cudaMemcpyDeviceToHost, s), "d2h");
    check(cudaFreeAsync(d_ptr, s), "free");
    check(cudaFreeAsync(d_perm, s), "free");
    check(cudaStreamSynchronize(s), "nnz_sort sync");
  });
}

int parac_gpu_upload(parac_gpu_ctx* ctx, const parac_csr* g, const int32_t* perm) {
  NvtxRange nvtx_range("parac_gpu_upload");
  return guarded([&] {
    require_ctx(ctx);
    if (!g || g->n < 0 || !g->ptr) throw Failure{dimension_mismatch, "bad graph"};
    const int n = g->n;
    const long long nnz = g->ptr[n];
    if (n > 0 && !perm) throw Failure{dimension_mismatch, "null ordering"};
    // nothing staged is valid until every copy below has succeeded
    ctx->n = -1;
    ctx->f_n = -1;
    ctx->batch_count = 0;
    solve_invalidate(ctx->solve);
    ctx->ptr.ensure(static_cast<std::size_t>(n) + 1);
    ctx->adj.ensure(static_cast<std::size_t>(std::max<long long>(nnz, 1)));
    ctx->w.ensure(static_cast<std::size_t>(std::max<long long>(nnz, 1)));
    ctx->perm.ensure(static_cast<std::size_t>(std::max(n, 1)));
    cudaStream_t s = ctx->stream;
    ctx->stage.h2d(ctx->ptr.p, g->ptr, sizeof(long long) * (n + 1), s);
    if (nnz > 0) {
      ctx->stage.h2d(ctx->adj.p, g->adj, sizeof(int) * nnz, s);
      ctx->stage.h2d(ctx->w.p, g->w, sizeof(double) * nnz, s);
    }
    if (n > 0) ctx->stage.h2d(ctx->perm.p, perm, sizeof(int) * n, s);
    ctx->scalar.ensure(1);
    max_degree_device(n, ctx->ptr.p, ctx->scalar.p, s, device_sms(ctx));
    check(cudaMemcpyAsync(&ctx->max_degree, ctx->scalar.p, sizeof(long long), cudaMemcpyDeviceToHost, s), "d2h");
    ctx->needs_hubs = false;
    check(cudaStreamSynchronize(s), "h2d sync");
    ctx->n = n;
    ctx->nnz = nnz;
    ctx->f_n = -1;
    ctx->batch_count = 0;
    solve_invalidate(ctx->solve);
  });
}

// Batch (BASELINE config[4]): stage `count` independent problems as ONE
// disjoint-union graph -- labels and positions of problem i are offset by the
// sizes of problems 0..i-1 -- so one persistent elimination kernel factors
// them all at once. Each position keeps its own problem's sample seed and
// local position as the RNG key, and fills never cross components, so every
// problem's factor is byte-identical to its stand-alone factorization.
int parac_gpu_upload_batch(parac_gpu_ctx* ctx, int32_t count, const parac_csr* graphs,
                           const int32_t* const* perms, const uint64_t* seeds) {
  NvtxRange nvtx_range("parac_gpu_upload_batch");
  return guarded([&] {
    require_ctx(ctx);
    if (count <= 0 || !graphs || !perms || !seeds) throw Failure{dimension_mismatch, "empty batch"};
    ctx->n = -1;
    ctx->f_n = -1;
    ctx->batch_count = 0;
    solve_invalidate(ctx->solve);
    // every member's ordering must be a permutation of its own [0, n_i): the
    // union check on the device cannot tell a valid union of invalid members
    long long total_n = 0;
    for (int i = 0; i < count; ++i) {
      const int ni = graphs[i].n;
      if (ni < 0 || !graphs[i].ptr || (ni > 0 && !perms[i])) throw Failure{dimension_mismatch, "bad graph in batch"};
      total_n += ni;
    }
    {  // members checked side by side on host threads; the lowest failing member is reported
      std::vector<int> bad_v(static_cast<std::size_t>(count), -1);
      auto check_member = [&](int i) {
        const int ni = graphs[i].n;
        std::vector<unsigned char> seen(static_cast<std::size_t>(ni), 0);
        for (int v = 0; v < ni; ++v) {
          const int q = perms[i][v];
          if (q < 0 || q >= ni || seen[q]) {
            bad_v[i] = v;
            return;
          }
          seen[q] = 1;
        }
      };
      const int nt = total_n >= (1 << 20)
                         ? static_cast<int>(std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 16u))
                         : 1;
      if (nt <= 1 || count == 1) {
        for (int i = 0; i < count; ++i) check_member(i);
      } else {
        std::atomic<int> next{0};
        std::vector<std::thread> th;
        for (int t = 0; t < std::min(nt, count); ++t)
          th.emplace_back([&] {
            for (int i; (i = next.fetch_add(1)) < count;) check_member(i);
          });
        for (auto& t : th) t.join();
      }
      for (int i = 0; i < count; ++i)
        if (bad_v[i] >= 0)
          throw Failure{not_a_permutation, "ordering of batch problem " + std::to_string(i) +
                                               " is not a permutation (vertex " + std::to_string(bad_v[i]) + ")"};
    }
    long long N = 0, NNZ = 0;
    std::vector<long long> base(static_cast<std::size_t>(count) + 1, 0), ebase(base);
    std::vector<unsigned long long> ps(static_cast<std::size_t>(count));
    for (int i = 0; i < count; ++i) {
      if (graphs[i].n < 0) throw Failure{dimension_mismatch, "bad graph in batch"};
      base[i] = N;
      ebase[i] = NNZ;
      N += graphs[i].n;
      NNZ += graphs[i].ptr[graphs[i].n];
      ps[i] = derive_seed(seeds[i], kSaltSampling);
    }
    base[count] = N;
    ebase[count] = NNZ;
    if (N > 2147483647LL) throw Failure{dimension_mismatch, "batch exceeds 2^31 vertices"};
    // Problems are copied straight into their slices of the device union (from
    // the caller's buffers; pinned memory copies at full PCIe/C2C rate), then
    // one pass adds the label / edge offsets on the device.
    cudaStream_t s = ctx->stream;
    const std::size_t nn = static_cast<std::size_t>(std::max<long long>(N, 1));
    const std::size_t ee = static_cast<std::size_t>(std::max<long long>(NNZ, 1));
    ctx->ptr.ensure(nn + 1);
    ctx->adj.ensure(ee);
    ctx->w.ensure(ee);
    ctx->perm.ensure(nn);
    ctx->pos_pid.ensure(nn);
    ctx->pid_base.ensure(static_cast<std::size_t>(count) + 1);
    ctx->pid_ebase.ensure(static_cast<std::size_t>(count) + 1);
    ctx->pid_seed.ensure(static_cast<std::size_t>(count));
    for (int i = 0; i < count; ++i) {
      const parac_csr& g = graphs[i];
      const long long m = g.ptr[g.n];
      check(cudaMemcpyAsync(ctx->ptr.p + base[i], g.ptr, sizeof(long long) * g.n, cudaMemcpyHostToDevice, s), "h2d");
      if (m > 0) {
        check(cudaMemcpyAsync(ctx->adj.p + ebase[i], g.adj, sizeof(int) * m, cudaMemcpyHostToDevice, s), "h2d");
        check(cudaMemcpyAsync(ctx->w.p + ebase[i], g.w, sizeof(double) * m, cudaMemcpyHostToDevice, s), "h2d");
      }
      if (g.n > 0)
        check(cudaMemcpyAsync(ctx->perm.p + base[i], perms[i], sizeof(int) * g.n, cudaMemcpyHostToDevice, s), "h2d");
    }
    check(cudaMemcpyAsync(ctx->pid_base.p, base.data(), sizeof(long long) * (count + 1), cudaMemcpyHostToDevice, s), "h2d");
    check(cudaMemcpyAsync(ctx->pid_ebase.p, ebase.data(), sizeof(long long) * (count + 1), cudaMemcpyHostToDevice, s), "h2d");
    check(cudaMemcpyAsync(ctx->pid_seed.p, ps.data(), sizeof(unsigned long long) * count, cudaMemcpyHostToDevice, s), "h2d");
    check(launch_batch_offsets(count, N, NNZ, ctx->pid_base.p, ctx->pid_ebase.p, ctx->ptr.p, ctx->adj.p,
                               ctx->perm.p, ctx->pos_pid.p, s), "batch offsets");
    ctx->scalar.ensure(1);
    max_degree_device(static_cast<int>(N), ctx->ptr.p, ctx->scalar.p, s, device_sms(ctx));
    check(cudaMemcpyAsync(&ctx->max_degree, ctx->scalar.p, sizeof(long long), cudaMemcpyDeviceToHost, s), "d2h");
    ctx->needs_hubs = false;
    check(cudaStreamSynchronize(s), "h2d sync");
    ctx->n = static_cast<int>(N);
    ctx->nnz = NNZ;
    ctx->f_n = -1;
    solve_invalidate(ctx->solve);
    ctx->batch_count = count;
    ctx->batch_base_h = base;
    // streamer blocks (stream_assemble.cu): up to kStreamBlock positions, never across problems
    ctx->blk_k0_h.clear();
    for (int i = 0; i < count; ++i)
      for (long long k = base[i]; k < base[i + 1]; k += kStreamBlock) ctx->blk_k0_h.push_back(static_cast<int>(k));
    ctx->blk_k0_h.push_back(static_cast<int>(N));
    ctx->blk_k0.ensure(ctx->blk_k0_h.size());
    check(cudaMemcpy(ctx->blk_k0.p, ctx->blk_k0_h.data(), sizeof(int) * ctx->blk_k0_h.size(), cudaMemcpyHostToDevice),
          "h2d");
    const int nblk = static_cast<int>(ctx->blk_k0_h.size()) - 1;
    ctx->blk_mem_h.assign(nblk, 0);
    ctx->blk_first_h.assign(nblk, 0);
    std::vector<int> mfirst(count, -1), mcount(count, 0);
    for (int b = 0, p = 0; b < nblk; ++b) {
      while (ctx->blk_k0_h[b] >= base[p + 1]) ++p;
      if (mfirst[p] < 0) mfirst[p] = b;
      ctx->blk_mem_h[b] = p;
      ctx->blk_first_h[b] = mfirst[p];
      ++mcount[p];
    }
    ctx->claim_h.clear();  // j-th block of every member, then the (j+1)-th: members progress side by side
    for (int j = 0, more = 1; more; ++j) {
      more = 0;
      for (int p = 0; p < count; ++p)
        if (j < mcount[p]) {
          ctx->claim_h.push_back(mfirst[p] + j);
          more = 1;
        }
    }
    ctx->blk_first.ensure(std::max(nblk, 1));
    ctx->claim.ensure(std::max(nblk, 1));
    if (nblk > 0) {
      check(cudaMemcpy(ctx->blk_first.p, ctx->blk_first_h.data(), sizeof(int) * nblk, cudaMemcpyHostToDevice), "h2d");
      check(cudaMemcpy(ctx->claim.p, ctx->claim_h.data(), sizeof(int) * nblk, cudaMemcpyHostToDevice), "h2d");
    }
    ctx->batch_ebase_h = ebase;
    ctx->batch_regions = false;
  });
}

int parac_gpu_factor_batch(parac_gpu_ctx* ctx, int32_t count, const parac_csr* graphs,
                           const int32_t* const* perms, const uint64_t* seeds, const parac_gpu_options* opt,
                           parac_gpu_factor_info* info) {
  Timer wall;
  int rc = parac_gpu_upload_batch(ctx, count, graphs, perms, seeds);
  if (rc) return rc;
  const double up = wall.ms();
  rc = parac_gpu_factor_resident(ctx, 0, opt, info);
  if (rc == 0 && info) {
    info->upload_ms = up;
    info->wall_ms = wall.ms();
  }
  return rc;
}

int parac_gpu_batch_nnz(parac_gpu_ctx* ctx, int32_t i, int64_t* nnz_off) {
  return guarded([&] {
    require_ctx(ctx);
    if (ctx->f_n < 0 || ctx->batch_count <= 0 || i < 0 || i >= ctx->batch_count)
      throw Failure{dimension_mismatch, "no resident batch factor / index out of range"};
    if (ctx->batch_regions) {
      *nnz_off = ctx->batch_z_h[i];
      return;
    }
    long long c[2];
    const long long b = ctx->batch_base_h[i], e = ctx->batch_base_h[i + 1];
    check(cudaMemcpy(&c[0], ctx->col_ptr.p + b, sizeof(long long), cudaMemcpyDeviceToHost), "d2h");
    check(cudaMemcpy(&c[1], ctx->col_ptr.p + e, sizeof(long long), cudaMemcpyDeviceToHost), "d2h");
    *nnz_off = c[1] - c[0];
  });
}

int parac_gpu_download_batch(parac_gpu_ctx* ctx, int32_t i, int64_t* col_ptr, int32_t* rows, double* values,
                             double* diag) {
  NvtxRange nvtx_range("parac_gpu_download_batch");
  return guarded([&] {
    require_ctx(ctx);
    if (ctx->f_n < 0 || ctx->batch_count <= 0 || i < 0 || i >= ctx->batch_count)
      throw Failure{dimension_mismatch, "no resident batch factor / index out of range"};
    const long long b = ctx->batch_base_h[i], e = ctx->batch_base_h[i + 1];
    const long long n = e - b;
    cudaStream_t s = ctx->stream;
    if (ctx->batch_regions) {  // streamed: member i's local col_ptr and its region
      const long long z = ctx->batch_z_h[i], r0 = ctx->region_h[i];
      if (col_ptr) check(cudaMemcpyAsync(col_ptr, ctx->lcol.p + b + i, sizeof(long long) * (n + 1), cudaMemcpyDeviceToHost, s), "d2h");
      if (rows && z) check(cudaMemcpyAsync(rows, ctx->rows.p + r0, sizeof(int) * z, cudaMemcpyDeviceToHost, s), "d2h");
      if (values && z) check(cudaMemcpyAsync(values, ctx->vals.p + r0, sizeof(double) * z, cudaMemcpyDeviceToHost, s), "d2h");
      if (diag && n) check(cudaMemcpyAsync(diag, ctx->diag.p + b, sizeof(double) * n, cudaMemcpyDeviceToHost, s), "d2h");
      check(cudaStreamSynchronize(s), "d2h sync");
      if (!col_ptr) return;
      if (n == 0) col_ptr[0] = 0;
      return;
    }
    check(cudaMemcpyAsync(col_ptr, ctx->col_ptr.p + b, sizeof(long long) * (n + 1), cudaMemcpyDeviceToHost, s), "d2h");
    check(cudaStreamSynchronize(s), "d2h sync");
    const long long z0 = col_ptr[0], z = col_ptr[n] - z0;
    if (rows && z) check(cudaMemcpyAsync(rows, ctx->rows.p + z0, sizeof(int) * z, cudaMemcpyDeviceToHost, s), "d2h");
    if (values && z) check(cudaMemcpyAsync(values, ctx->vals.p + z0, sizeof(double) * z, cudaMemcpyDeviceToHost, s), "d2h");
    if (diag && n) check(cudaMemcpyAsync(diag, ctx->diag.p + b, sizeof(double) * n, cudaMemcpyDeviceToHost, s), "d2h");
    check(cudaStreamSynchronize(s), "d2h sync");
    for (long long k = 0; k <= n; ++k) col_ptr[k] -= z0;  // rows were made local on the device
  });
}

int parac_gpu_factor_begin(parac_gpu_ctx* ctx, uint64_t seed, const parac_gpu_options* opt) {
  NvtxRange nvtx_range("parac_gpu_factor_begin");
  parac_gpu_options o;
  if (opt) o = *opt; else parac_gpu_default_options(&o);
  return guarded([&] {
    require_ctx(ctx);
    if (ctx->n < 0) throw Failure{dimension_mismatch, "no graph staged (call parac_gpu_upload)"};
    if (ctx->pending) throw Failure{internal_error, "a factorization is pending (call parac_gpu_factor_end)"};
    // the previous resident factor is gone as soon as its buffers are reused
    ctx->f_n = -1;
    solve_invalidate_factor(ctx->solve);
    ctx->p_t0 = std::chrono::steady_clock::now();
    ctx->p_seed = seed;
    ctx->p_opt = o;
    ctx->p_b = default_budgets(ctx->n, ctx->nnz / 2, ctx->max_degree, o, ctx->pool0.cap * sizeof(int4));
    ctx->p_attempts = 0;
    ctx->p_failed_ms = 0.0;
    ctx->streaming = stream_wanted(ctx);
    launch_factor(ctx, seed, o, ctx->p_b);
    ctx->pending = true;
  });
}

}  // extern "C"

namespace {
// parac_gpu_factor_end / parac_gpu_factor_batch_end: one problem's outputs
// (hout) or every batch member's (bout), either may be null.
int factor_end_impl(parac_gpu_ctx* ctx, parac_gpu_factor_info* info, const HostOut* hout, BatchOut* bout) {
  int rc = guarded([&] {
    require_ctx_any(ctx);
    if (!ctx->pending) throw Failure{internal_error, "no factorization pending (call parac_gpu_factor_begin)"};
  });
  if (rc) return rc;
  const HostOut out = hout ? *hout : HostOut{nullptr, nullptr, nullptr, nullptr, 0};
  int64_t* const col_ptr = out.col_ptr;
  int32_t* const rows = out.rows;
  double* const values = out.values;
  double* const diag = out.diag;
  const long long capacity = out.cap;
  const bool want = col_ptr || rows || values || diag;
  const parac_gpu_options& o = ctx->p_opt;
  Budgets& b = ctx->p_b;
  const int n = ctx->n;
  const long long E = ctx->nnz / 2;
  for (;;) {
    int st = 0;
    rc = guarded([&] { st = complete_factor(ctx, o, b, want ? &out : nullptr, bout); });
    if (rc) {
      ctx->pending = false;
      return rc;
    }
    ++ctx->p_attempts;
    if (st == 0) break;
    {
      float t = 0;
      if (cudaEventSynchronize(ctx->ev[3]) == cudaSuccess && cudaEventElapsedTime(&t, ctx->ev[0], ctx->ev[3]) == cudaSuccess)
        ctx->p_failed_ms += t;
      if (std::getenv("PARAC_VERBOSE"))
        std::fprintf(stderr, "parac_gpu: attempt %d ran out of budget after %.1f ms: %s\n", ctx->p_attempts - 1, t,
                     last_error());
    }
    // Budget exhaustion with library-chosen budgets: grow and retry (the
    // caller's explicit budgets fail cleanly, like ParOptions::arena_budget).
    const bool defaults = o.fill_pool_entries < 0 && o.column_arena_entries < 0;
    bool again = false;
    if (st == kStatusNeedHubs && ctx->p_attempts <= 8) {
      again = true;  // now with the hub path
    } else if (st == arena_exhausted && defaults && ctx->p_attempts <= 4) {
      b.ovf *= 2;
      b.arena *= 2;
      b.large *= 4;
      again = true;
    }
    if (!again) {
      ctx->pending = false;
      return st;
    }
    rc = guarded([&] { launch_factor(ctx, ctx->p_seed, o, b); });
    if (rc) {
      ctx->pending = false;
      return rc;
    }
  }
  ctx->pending = false;
  rc = guarded([&] {
    if (ctx->streaming && ctx->batch_count > 0) {  // member regions (stream_assemble.cu)
      int ov = 0;
      check(cudaMemcpy(&ov, ctx->overflow.p, sizeof(int), cudaMemcpyDeviceToHost), "d2h");
      if (ov) {  // a member outgrew its region: the union CSC after all, assembled now
        FactorDev d{};
        d.n = n;
        d.col_len = ctx->col_len.p;
        d.col_start = ctx->col_start.p;
        d.arena_rows = ctx->arena_rows.p;
        d.arena_vals = ctx->arena_vals.p;
        d.samples = ctx->samples.p;
        d.ctrl = ctx->ctrl.p;  // (its total_fills was read already)
        check(launch_assemble(d, ctx->col_ptr.p, ctx->rows.p, ctx->vals.p, ctx->tiles.p, ctx->stream), "assemble");
        check(launch_batch_local_rows(n, ctx->col_ptr.p, ctx->pos_pid.p, ctx->pid_base.p, ctx->rows.p, ctx->stream),
              "batch rows");
        check(cudaMemcpyAsync(&ctx->last_z, ctx->col_ptr.p + n, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream),
              "d2h");
        check(cudaStreamSynchronize(ctx->stream), "assemble sync");
        ctx->batch_regions = false;
        if (bout) bout->redo = true;
      } else {
        const int count = ctx->batch_count;
        ctx->batch_z_h.assign(count, 0);
        for (int b = 0, nb = static_cast<int>(ctx->blk_mem_h.size()); b < nb; ++b)  // the member's last block's word
          ctx->batch_z_h[ctx->blk_mem_h[b]] = static_cast<long long>(ctx->blkh_h[b] & ~(1ull << 63));
        long long Zs = 0;
        for (long long z : ctx->batch_z_h) Zs += z;
        ctx->last_z = Zs;
        ctx->batch_regions = true;
      }
    } else {
      ctx->batch_regions = false;
    }
    const Ctrl c = ctx->last_ctrl;
    const long long Z = ctx->last_z;
    ctx->f_n = n;
    ctx->f_nnz = Z;
    ctx->f_has_stats = true;
    ctx->f_external = false;
    if (ctx->batch_count > 0 && !ctx->streaming) {  // each problem's rows in its own position space (the streamer did it)
      check(launch_batch_local_rows(n, ctx->col_ptr.p, ctx->pos_pid.p, ctx->pid_base.p, ctx->rows.p, ctx->stream),
            "batch rows");
      check(cudaStreamSynchronize(ctx->stream), "batch rows sync");
    }
    solve_invalidate_factor(ctx->solve);
    if (info) {
      std::memset(info, 0, sizeof(*info));
      info->n = n;
      info->num_edges = E;
      info->nnz_off_diagonal = Z;
      info->total_fills = c.total_fills;
      info->fill_pool_used = static_cast<long long>(c.ovf_bump);
      info->arena_used = Z;
      info->max_raw = c.max_raw;
      info->large_columns = c.large_cols;
      float t01 = 0, t12 = 0, t23 = 0, t03 = 0;
      cudaEventElapsedTime(&t01, ctx->ev[0], ctx->ev[1]);
      cudaEventElapsedTime(&t12, ctx->ev[1], ctx->ev[2]);
      cudaEventElapsedTime(&t23, ctx->ev[2], ctx->ev[3]);
      cudaEventElapsedTime(&t03, ctx->ev[0], ctx->ev[3]);
      info->setup_ms = t01;
      info->eliminate_ms = t12;
      info->assemble_ms = t23;
      info->device_ms = t03 + ctx->p_failed_ms;
      info->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ctx->p_t0).count();
      info->attempts = ctx->p_attempts;
    }
    if (want && Z > capacity && (rows || values))
      throw Failure{budget_exceeded, "factor has " + std::to_string(Z) + " off-diagonal entries, outputs hold " +
                                         std::to_string(capacity) + " (the factor stays resident: parac_gpu_download)"};
    if (want && !ctx->streaming) {  // the assembly ran after K3: plain download
      const long long z = std::min<long long>(Z, std::max<long long>(capacity, 0));
      if (col_ptr) ctx->stage.d2h(col_ptr, ctx->col_ptr.p, sizeof(long long) * (n + 1), ctx->stream);
      if (rows && z) ctx->stage.d2h(rows, ctx->rows.p, sizeof(int) * z, ctx->stream);
      if (values && z) ctx->stage.d2h(values, ctx->vals.p, sizeof(double) * z, ctx->stream);
      if (diag && n) ctx->stage.d2h(diag, ctx->diag.p, sizeof(double) * n, ctx->stream);
      check(cudaStreamSynchronize(ctx->stream), "d2h sync");
    }
    if (bout && (!ctx->streaming || bout->redo)) {  // assembled after K3: every member's copies in flight at once
      bout->short_cap = false;
      ensure_stream_resources(ctx);
      const int count = ctx->batch_count;
      const std::vector<long long>& base = ctx->batch_base_h;
      std::vector<long long> zb(static_cast<std::size_t>(count) + 1);
      for (int i = 0; i <= count; ++i)  // each member's first entry offset (and the total)
        check(cudaMemcpyAsync(&zb[i], ctx->col_ptr.p + base[i], sizeof(long long), cudaMemcpyDeviceToHost, ctx->s_copy),
              "d2h");
      check(cudaStreamSynchronize(ctx->s_copy), "d2h sync");
      for (int i = 0; i < count; ++i) {
        const long long z0 = zb[i], z = zb[i + 1] - z0, m = base[i + 1] - base[i];
        const bool fits = !bout->caps || z <= bout->caps[i];
        if (!fits) bout->short_cap = true;
        if (bout->col_ptr && bout->col_ptr[i])
          copy_range(ctx, bout->col_ptr[i], ctx->col_ptr.p + base[i], sizeof(long long) * (m + 1));
        if (fits && bout->rows && bout->rows[i]) copy_range(ctx, bout->rows[i], ctx->rows.p + z0, sizeof(int) * z);
        if (fits && bout->values && bout->values[i])
          copy_range(ctx, bout->values[i], ctx->vals.p + z0, sizeof(double) * z);
        if (bout->diag && bout->diag[i]) copy_range(ctx, bout->diag[i], ctx->diag.p + base[i], sizeof(double) * m);
      }
      check(cudaStreamSynchronize(ctx->s_copy), "d2h sync");
      if (bout->col_ptr) {  // local column pointers (rows were made local on the device), members on threads
        std::atomic<int> next{0};
        auto work = [&] {
          for (int i; (i = next.fetch_add(1)) < count;) {
            std::int64_t* cp = bout->col_ptr[i];
            if (!cp) continue;
            for (long long k = 0, m = base[i + 1] - base[i]; k <= m; ++k) cp[k] -= zb[i];
          }
        };
        const int nt = static_cast<int>(std::min<long long>(std::min(count, 8), std::max<long long>(1, ctx->n >> 20)));
        std::vector<std::thread> th;
        for (int t = 1; t < nt; ++t) th.emplace_back(work);
        work();
        for (auto& t : th) t.join();
      }
    }
    if (bout && bout->short_cap)
      throw Failure{budget_exceeded, "a batch member's factor exceeds its output capacity (the factor stays "
                                     "resident: parac_gpu_batch_nnz + parac_gpu_download_batch)"};
  });
  return rc;
}
}  // namespace

extern "C" {

int parac_gpu_factor_end(parac_gpu_ctx* ctx, parac_gpu_factor_info* info, int64_t* col_ptr, int32_t* rows,
                         double* values, double* diag, int64_t capacity) {
  NvtxRange nvtx_range("parac_gpu_factor_end");
  const bool want = col_ptr || rows || values || diag;
  if (want && ctx && ctx->batch_count > 0) {
    const int rc = factor_end_impl(ctx, info, nullptr, nullptr);  // complete it; the outputs do not apply
    if (rc) return rc;
    return guarded([] { throw Failure{dimension_mismatch, "a batch is staged: use parac_gpu_factor_batch_end"}; });
  }
  const HostOut out{col_ptr, rows, values, diag, capacity};
  return factor_end_impl(ctx, info, &out, nullptr);
}

int parac_gpu_factor_batch_end(parac_gpu_ctx* ctx, parac_gpu_factor_info* info, int64_t* const* col_ptrs,
                               int32_t* const* rows, double* const* values, double* const* diags,
                               const int64_t* capacities) {
  NvtxRange nvtx_range("parac_gpu_factor_batch_end");
  if (ctx && ctx->pending && ctx->batch_count <= 0) {
    const int rc = factor_end_impl(ctx, info, nullptr, nullptr);
    if (rc) return rc;
    return guarded([] { throw Failure{dimension_mismatch, "no batch staged: use parac_gpu_factor_end"}; });
  }
  BatchOut out{col_ptrs, rows, values, diags, capacities};
  const bool want = col_ptrs || rows || values || diags;
  return factor_end_impl(ctx, info, nullptr, want ? &out : nullptr);
}

int parac_gpu_factor_batch_to_host(parac_gpu_ctx* ctx, int32_t count, const parac_csr* graphs,
                                   const int32_t* const* perms, const uint64_t* seeds, const parac_gpu_options* opt,
                                   parac_gpu_factor_info* info, int64_t* const* col_ptrs, int32_t* const* rows,
                                   double* const* values, double* const* diags, const int64_t* capacities) {
  const auto t0 = std::chrono::steady_clock::now();
  int rc = parac_gpu_upload_batch(ctx, count, graphs, perms, seeds);
  if (rc) return rc;
  const double up = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  rc = parac_gpu_factor_begin(ctx, 0, opt);
  if (rc) return rc;
  rc = parac_gpu_factor_batch_end(ctx, info, col_ptrs, rows, values, diags, capacities);
  if (info && (rc == 0 || rc == budget_exceeded)) {
    info->upload_ms = up;
    info->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return rc;
}

int parac_gpu_factor_resident(parac_gpu_ctx* ctx, uint64_t seed, const parac_gpu_options* opt,
                              parac_gpu_factor_info* info) {
  const int rc = parac_gpu_factor_begin(ctx, seed, opt);
  if (rc) return rc;
  return parac_gpu_factor_end(ctx, info, nullptr, nullptr, nullptr, nullptr, 0);
}

int parac_gpu_factor_to_host(parac_gpu_ctx* ctx, const parac_csr* g, const int32_t* perm, uint64_t seed,
                             const parac_gpu_options* opt, parac_gpu_factor_info* info, int64_t* col_ptr,
                             int32_t* rows, double* values, double* diag, int64_t capacity) {
  const auto t0 = std::chrono::steady_clock::now();
  int rc = parac_gpu_upload(ctx, g, perm);
  if (rc) return rc;
  const double up = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  rc = parac_gpu_factor_begin(ctx, seed, opt);
  if (rc) return rc;
  rc = parac_gpu_factor_end(ctx, info, col_ptr, rows, values, diag, capacity);
  if (info && (rc == 0 || rc == budget_exceeded)) {
    info->upload_ms = up;
    info->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return rc;
}

int parac_gpu_factor(parac_gpu_ctx* ctx, const parac_csr* g, const int32_t* perm, uint64_t seed,
                     const parac_gpu_options* opt, parac_gpu_factor_info* info) {
  Timer wall;
  int rc = parac_gpu_upload(ctx, g, perm);
  if (rc) return rc;
  const double up = wall.ms();
  rc = parac_gpu_factor_resident(ctx, seed, opt, info);
  if (rc == 0 && info) {
    info->upload_ms = up;
    info->wall_ms = wall.ms();
  }
  return rc;
}

int parac_gpu_download(parac_gpu_ctx* ctx, int64_t* col_ptr, int32_t* rows, double* values,
                       double* diag, int32_t* merged_degree, int32_t* samples_emitted,
                       int32_t* fills_received) {
  NvtxRange nvtx_range("parac_gpu_download");
  return guarded([&] {
    require_ctx(ctx);
    if (ctx->f_n < 0) throw Failure{dimension_mismatch, "no resident factor"};
    if (ctx->batch_count > 0 && ctx->batch_regions)
      throw Failure{dimension_mismatch, "the resident factor is a streamed batch: parac_gpu_download_batch"};
    const int n = ctx->f_n;
    const long long Z = ctx->f_nnz;
    cudaStream_t s = ctx->stream;
    if (col_ptr) ctx->stage.d2h(col_ptr, ctx->col_ptr.p, sizeof(long long) * (n + 1), s);
    if (rows && Z) ctx->stage.d2h(rows, ctx->rows.p, sizeof(int) * Z, s);
    if (values && Z) ctx->stage.d2h(values, ctx->vals.p, sizeof(double) * Z, s);
    const double* dsrc = ctx->f_external ? ctx->f_diag_ext.p : ctx->diag.p;
    if (diag && n) ctx->stage.d2h(diag, dsrc, sizeof(double) * n, s);
    if ((merged_degree || samples_emitted || fills_received) && !ctx->f_has_stats)
      throw Failure{internal_error, "factor has no device stats (uploaded externally)"};
    if (merged_degree && n) ctx->stage.d2h(merged_degree, ctx->col_len.p, sizeof(int) * n, s);
    if (samples_emitted && n) ctx->stage.d2h(samples_emitted, ctx->samples.p, sizeof(int) * n, s);
    if (fills_received && n) {
      ctx->heavy_list.ensure(static_cast<std::size_t>(std::max(n, 1)));  // scratch (K1 only uses it earlier)
      check(launch_extract_fills(n, ctx->cnt.p, ctx->heavy_list.p, s), "fills");
      ctx->stage.d2h(fills_received, ctx->heavy_list.p, sizeof(int) * n, s);
    }
    check(cudaStreamSynchronize(s), "d2h sync");
  });
}

int parac_gpu_upload_factor(parac_gpu_ctx* ctx, int32_t n, const int64_t* col_ptr,
                            const int32_t* rows, const double* values, const double* diag,
                            const int32_t* perm) {
  NvtxRange nvtx_range("parac_gpu_upload_factor");
  return guarded([&] {
    require_ctx(ctx);
    // The sweeps trust the factor's structure (levels are built by waiting on
    // earlier columns), so a malformed factor is rejected here, before any
    // device work: the reference's apply_preconditioner would just read it.
    if (n < 0 || !col_ptr || (n > 0 && (!diag || !perm)))
      throw Failure{dimension_mismatch, "bad factor arrays"};
    if (col_ptr[0] != 0) throw Failure{dimension_mismatch, "factor col_ptr[0] != 0"};
    for (int k = 0; k < n; ++k)
      if (col_ptr[k + 1] < col_ptr[k]) throw Failure{dimension_mismatch, "factor col_ptr is not monotone"};
    const long long Z = col_ptr[n];
    if (Z > 0 && (!rows || !values)) throw Failure{dimension_mismatch, "bad factor arrays"};
    for (int k = 0; k < n; ++k)
      for (long long p = col_ptr[k]; p < col_ptr[k + 1]; ++p)
        if (rows[p] <= k || rows[p] >= n)
          throw Failure{dimension_mismatch, "factor row " + std::to_string(rows[p]) + " of column " +
                                                std::to_string(k) + " is not strictly below the diagonal"};
    {
      std::vector<unsigned char> seen(static_cast<std::size_t>(n), 0);
      for (int v = 0; v < n; ++v) {
        const int q = perm[v];
        if (q < 0 || q >= n || seen[q]) throw Failure{not_a_permutation, "factor perm is not a permutation"};
        seen[q] = 1;
      }
    }
    ctx->f_n = -1;  // published only after every copy succeeded
    solve_invalidate_factor(ctx->solve);
    cudaStream_t s = ctx->stream;
    ctx->col_ptr.ensure(static_cast<std::size_t>(n) + 1);
    ctx->rows.ensure(static_cast<std::size_t>(std::max<long long>(Z, 1)));
    ctx->vals.ensure(static_cast<std::size_t>(std::max<long long>(Z, 1)));
    ctx->f_diag_ext.ensure(static_cast<std::size_t>(std::max(n, 1)));
    ctx->f_perm_ext.ensure(static_cast<std::size_t>(std::max(n, 1)));
    ctx->stage.h2d(ctx->col_ptr.p, col_ptr, sizeof(long long) * (n + 1), s);
    if (Z) {
      ctx->stage.h2d(ctx->rows.p, rows, sizeof(int) * Z, s);
      ctx->stage.h2d(ctx->vals.p, values, sizeof(double) * Z, s);
    }
    if (n) {
      ctx->stage.h2d(ctx->f_diag_ext.p, diag, sizeof(double) * n, s);
      ctx->stage.h2d(ctx->f_perm_ext.p, perm, sizeof(int) * n, s);
    }
    check(cudaStreamSynchronize(s), "h2d sync");
    ctx->f_n = n;
    ctx->f_nnz = Z;
    ctx->f_has_stats = false;
    ctx->f_external = true;
    if (ctx->batch_count > 0) {  // an uploaded factor replaces a resident batch; the
      ctx->batch_count = 0;      // staged union graph means nothing without it
      ctx->n = -1;
      solve_invalidate(ctx->solve);
    }
    solve_invalidate_factor(ctx->solve);
  });
}

int parac_gpu_download_times(parac_gpu_ctx* ctx, uint64_t* start_end) {
  return guarded([&] {
    require_ctx(ctx);
    if (!ctx->has_times || ctx->f_n < 0) throw Failure{internal_error, "no recorded times"};
    check(cudaMemcpy(start_end, ctx->vtimes.p, sizeof(unsigned long long) * 8 * ctx->f_n,
                     cudaMemcpyDeviceToHost), "d2h");
  });
}

int parac_gpu_download_subtimes(parac_gpu_ctx* ctx, uint64_t* sub) {
  return guarded([&] {
    require_ctx(ctx);
    if (!ctx->has_times || ctx->f_n < 0) throw Failure{internal_error, "no recorded times"};
    check(cudaMemcpy(sub, ctx->vsub.p, sizeof(unsigned long long) * 12 * ctx->f_n, cudaMemcpyDeviceToHost), "d2h");
  });
}

int parac_gpu_download_hub_trace(parac_gpu_ctx* ctx, uint64_t* out, int32_t cap, int32_t* count) {
  return guarded([&] {
    require_ctx(ctx);
    if (!ctx->has_times || ctx->f_n < 0) throw Failure{internal_error, "no recorded times"};
    const int cols = std::min(ctx->last_ctrl.large_cols, kHubTraceCap);
    if (count) *count = cols;
    const int c = std::min(cols, std::max(cap, 0));
    if (out && c > 0)
      check(cudaMemcpy(out, ctx->hub_trace.p, sizeof(unsigned long long) * kHubTraceWords * c, cudaMemcpyDeviceToHost),
            "d2h");
  });
}

int parac_gpu_download_phase_snapshots(parac_gpu_ctx* ctx, int64_t* dp, int32_t* taken) {
  return guarded([&] {
    require_ctx(ctx);
    if (ctx->trace_n < 0 || ctx->f_n < 0) throw Failure{internal_error, "no traced factor run"};
    if (dp)
      check(cudaMemcpy(dp, ctx->trace_dp.p, sizeof(long long) * 3 * ctx->trace_n, cudaMemcpyDeviceToHost), "d2h");
    if (taken) check(cudaMemcpy(taken, ctx->trace_taken.p, sizeof(int) * 3, cudaMemcpyDeviceToHost), "d2h");
  });
}

void* parac_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, std::max<size_t>(bytes, 1)) != cudaSuccess) return nullptr;
  return p;
}
void parac_host_free(void* p) {
  if (p) cudaFreeHost(p);
}
}  // extern "C"

// Accessors used by the solve translation unit.
namespace parac_gpu {
SolveInputs solve_inputs(parac_gpu_ctx* ctx) {
  SolveInputs in{};
  in.n = ctx->n;
  in.ptr = ctx->ptr.p;
  in.adj = ctx->adj.p;
  in.w = ctx->w.p;
  in.f_n = ctx->f_n;
  in.f_nnz = ctx->f_nnz;
  in.col_ptr = ctx->col_ptr.p;
  in.rows = ctx->rows.p;
  in.vals = ctx->vals.p;
  in.diag = ctx->f_external ? ctx->f_diag_ext.p : ctx->diag.p;
  in.perm = ctx->f_external ? ctx->f_perm_ext.p : ctx->perm.p;
  in.level = ctx->f_external ? nullptr : ctx->level.p;
  in.batch = ctx->batch_count;
  in.stream = ctx->stream;
  in.device = ctx->device;
  in.state = &ctx->solve;
  return in;
}
void ctx_activate(parac_gpu_ctx* ctx) { require_ctx(ctx); }
}  // namespace parac_gpu
