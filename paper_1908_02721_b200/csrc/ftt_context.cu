// Context, arena and error plumbing of the C ABI.
#include <stdarg.h>

#include <atomic>
#include <chrono>

#include <stdlib.h>

#include "ftt_common.cuh"

namespace ftt {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int arena_reserve(ftt_ctx *ctx, size_t bytes) {
  ctx->arena.used = 0;
  if (bytes <= ctx->arena.cap) return FTT_OK;
  size_t want = align_up(bytes + bytes / 4, 1 << 20);
  if (ctx->arena.base) {
    FTT_CUDA(cudaFreeAsync(ctx->arena.base, ctx->stream));
    ctx->arena.base = nullptr;
    ctx->arena.cap = 0;
  }
  void *p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, want, ctx->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    // retry with the exact size
    e = cudaMallocAsync(&p, align_up(bytes, 1 << 20), ctx->stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error("workspace allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
      return FTT_ERR_OOM;
    }
    want = align_up(bytes, 1 << 20);
  }
  ctx->arena.base = static_cast<char *>(p);
  ctx->arena.cap = want;
  return FTT_OK;
}

void *arena_take(ftt_ctx *ctx, size_t bytes) {
  bytes = align_up(bytes);
  if (ctx->arena.used + bytes > ctx->arena.cap) return nullptr;
  void *p = ctx->arena.base + ctx->arena.used;
  ctx->arena.used += bytes;
  return p;
}

// A few scalars to the host without the copy engine: one small kernel writes
// them into the context's pinned scratch (device-visible under UVA) and then
// a sequence word; the host spins on that word.  Against cudaMemcpyAsync +
// cudaStreamSynchronize this saves the DMA's start-up and the driver's wake
// (~6 us of each of the ~30 host round trips of a config-5 decomposition).
constexpr size_t kPostMax = 2048;   // bytes through k_post
constexpr size_t kPostFlag = 65536 - 64;  // the sequence word's offset in ctx->pinned

__global__ void k_post(const unsigned char *__restrict__ src, unsigned char *dst, unsigned bytes,
                       volatile unsigned *flag, unsigned seq) {
  const unsigned t = threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(src) | bytes) & 7) == 0) {
    for (unsigned i = t; i < bytes / 8; i += blockDim.x)
      reinterpret_cast<unsigned long long *>(dst)[i] =
          reinterpret_cast<const unsigned long long *>(src)[i];
  } else if (((reinterpret_cast<uintptr_t>(src) | bytes) & 3) == 0) {
    for (unsigned i = t; i < bytes / 4; i += blockDim.x)
      reinterpret_cast<unsigned *>(dst)[i] = reinterpret_cast<const unsigned *>(src)[i];
  } else {
    for (unsigned i = t; i < bytes; i += blockDim.x) dst[i] = src[i];
  }
  __threadfence_system();
  __syncthreads();
  if (t == 0) *flag = seq;
}

static int post_to_host(ftt_ctx *ctx, void *host, const void *dev, size_t bytes) {
  unsigned char *pin = static_cast<unsigned char *>(ctx->pinned);
  volatile unsigned *flag = reinterpret_cast<volatile unsigned *>(pin + kPostFlag);
  const unsigned seq = ++ctx->post_seq;
  k_post<<<1, 128, 0, ctx->stream>>>(static_cast<const unsigned char *>(dev), pin, (unsigned)bytes,
                                     flag, seq);
  FTT_LAUNCHED(ctx);
  for (unsigned spins = 1;; ++spins) {
    if (*flag == seq) break;
    if ((spins & 0x3fff) == 0) {  // a failed stream never sets the word
      const cudaError_t q = cudaStreamQuery(ctx->stream);
      if (q == cudaSuccess) {
        if (*flag == seq) break;
        set_error("post_to_host: the stream drained without the sequence word");
        return FTT_ERR_CUDA;
      }
      if (q != cudaErrorNotReady) {
        set_error("post_to_host: %s", cudaGetErrorString(q));
        return FTT_ERR_CUDA;
      }
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  memcpy(host, pin, bytes);
  return FTT_OK;
}

int copy_to_host(ftt_ctx *ctx, void *host, const void *dev, size_t bytes) {
  if (bytes == 0) return FTT_OK;
  struct Wait {
    ftt_ctx *c;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    ~Wait() {
      c->syncs++;
      c->sync_wait_ms +=
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  } wait{ctx};
  static const bool no_post = getenv("FTT_NO_POST") != nullptr;
  if (bytes <= kPostMax && !no_post) return post_to_host(ctx, host, dev, bytes);
  if (bytes <= kPostFlag) {
    FTT_CUDA(cudaMemcpyAsync(ctx->pinned, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    FTT_CUDA(cudaStreamSynchronize(ctx->stream));
    memcpy(host, ctx->pinned, bytes);
  } else {
    FTT_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    FTT_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return FTT_OK;
}

int copy_to_device(ftt_ctx *ctx, void *dev, const void *host, size_t bytes) {
  if (bytes == 0) return FTT_OK;
  if (bytes <= kPostFlag) {
    // the pinned scratch may still be read by an earlier async copy
    FTT_CUDA(cudaStreamSynchronize(ctx->stream));
    memcpy(ctx->pinned, host, bytes);
    FTT_CUDA(cudaMemcpyAsync(dev, ctx->pinned, bytes, cudaMemcpyHostToDevice, ctx->stream));
    FTT_CUDA(cudaStreamSynchronize(ctx->stream));
  } else {
    FTT_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    FTT_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return FTT_OK;
}

int stage_to_device(ftt_ctx *ctx, void *dev, const void *host, size_t bytes) {
  if (bytes == 0) return FTT_OK;
  const size_t b = align_up(bytes, 64);
  if (!ctx->ring || b > kRingBytes) {
    FTT_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    FTT_CUDA(cudaStreamSynchronize(ctx->stream));
    return FTT_OK;
  }
  if (ctx->ring_off + b > kRingBytes) {
    // wrap: every copy staged on the previous lap is done once the latest is
    FTT_CUDA(cudaEventSynchronize(ctx->ring_ev));
    ctx->ring_off = 0;
  }
  char *slot = ctx->ring + ctx->ring_off;
  ctx->ring_off += b;
  memcpy(slot, host, bytes);
  FTT_CUDA(cudaMemcpyAsync(dev, slot, bytes, cudaMemcpyHostToDevice, ctx->stream));
  FTT_CUDA(cudaEventRecord(ctx->ring_ev, ctx->stream));
  return FTT_OK;
}

int lin_chunks_wait_all(ftt_ctx *ctx) {
  const int n = ctx->lin_nchunks;
  ctx->lin_nchunks = 0;
  if (n > 0) FTT_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->lin_events[n - 1], 0));
  return FTT_OK;
}

int owned_alloc(ftt_ctx *ctx, void **p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) bytes = 256;
  cudaError_t e = cudaMallocAsync(p, bytes, ctx->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
    return FTT_ERR_OOM;
  }
  ctx->owned.push_back({*p, bytes});
  return FTT_OK;
}

int compact_status(ftt_ctx *ctx, size_t ntiles, uint64_t **status, unsigned **ticket,
                   uint32_t *epoch) {
  if (ntiles > ctx->cp_status_cap) {
    if (ctx->cp_status) FTT_CUDA(cudaFreeAsync(ctx->cp_status, ctx->stream));
    ctx->cp_status = nullptr;
    ctx->cp_status_cap = 0;
    const size_t cap = align_up(ntiles + ntiles / 4 + 64, 4096);
    FTT_CUDA(cudaMallocAsync((void **)&ctx->cp_status, 8 * (cap + 1), ctx->stream));
    FTT_CUDA(cudaMemsetAsync(ctx->cp_status, 0, 8 * (cap + 1), ctx->stream));
    ctx->cp_status_cap = cap;
    ctx->cp_epoch = 0;
  }
  // epochs 1 .. 2^30 - 1 tag the status words; on wrap the words are cleared
  if (++ctx->cp_epoch >= (1u << 30)) {
    FTT_CUDA(cudaMemsetAsync(ctx->cp_status, 0, 8 * ctx->cp_status_cap, ctx->stream));
    ctx->cp_epoch = 1;
  }
  *status = ctx->cp_status;
  *ticket = reinterpret_cast<unsigned *>(ctx->cp_status + ctx->cp_status_cap);
  *epoch = ctx->cp_epoch;
  return FTT_OK;
}

int zero_flags(ftt_ctx *ctx, size_t n, uint32_t **out) {
  if (n > ctx->zflags_cap) {
    if (ctx->zflags) FTT_CUDA(cudaFreeAsync(ctx->zflags, ctx->stream));
    ctx->zflags = nullptr;
    ctx->zflags_cap = 0;
    const size_t cap = align_up(n + n / 4, 1 << 20);
    FTT_CUDA(cudaMallocAsync((void **)&ctx->zflags, 4 * cap, ctx->stream));
    FTT_CUDA(cudaMemsetAsync(ctx->zflags, 0, 4 * cap, ctx->stream));
    ctx->zflags_cap = cap;
  }
  *out = ctx->zflags;
  return FTT_OK;
}

void owned_free(ftt_ctx *ctx, void *p) {
  if (!p) return;
  for (size_t i = 0; i < ctx->owned.size(); ++i) {
    if (ctx->owned[i].first == p) {
      cudaFreeAsync(p, ctx->stream);
      ctx->owned.erase(ctx->owned.begin() + i);
      return;
    }
  }
}

void svd_state_free(ftt_ctx *ctx);  // ftt_svd.cu

static int next_event(ftt_ctx *ctx) {
  if (ctx->ev_used >= (int)ctx->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    ctx->ev_pool.push_back(e);
  }
  return ctx->ev_used++;
}

int prof_begin(ftt_ctx *ctx) {
  if (!ctx->prof) return -1;
  int i = next_event(ctx);
  if (i >= 0) cudaEventRecord(ctx->ev_pool[i], ctx->stream);
  return i;
}

void prof_end(ftt_ctx *ctx, int begin, int tag, double bytes, double flops) {
  if (!ctx->prof || begin < 0) return;
  int i = next_event(ctx);
  if (i < 0) return;
  cudaEventRecord(ctx->ev_pool[i], ctx->stream);
  ctx->prof_recs.push_back({begin, i, tag, bytes, flops});
}

}  // namespace ftt

using namespace ftt;

extern "C" {

const char *ftt_version(void) { return "fasttt_b200 0.1.0 (sm_100a)"; }

const char *ftt_last_error(void) { return g_err; }

int ftt_create(int device, void *stream, ftt_ctx **ctx_out) {
  if (!ctx_out) {
    set_error("ctx_out is NULL");
    return FTT_ERR_INVALID;
  }
  *ctx_out = nullptr;
  FTT_CUDA(cudaSetDevice(device));
  ftt_ctx *ctx = new ftt_ctx();
  ctx->device = device;
  ctx->stream = static_cast<cudaStream_t>(stream);
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
    ctx->num_sms = sms;
  // Keep stream-ordered allocations cached in the device pool: the SVD
  // workspaces are allocated and released per truncation step, and with the
  // default release threshold (0) every step went back to the driver
  // (measured: per-step times varying 12..106 ms on config 2).
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      // Pre-grow the pool once: a decomposition's per-step buffers vary in
      // size, and a request that does not fit the pool's free space maps new
      // physical memory inside the call (measured ~2 ms per growth on
      // config 5, recurring as the pool fragments).  The block is freed at
      // once and stays reserved (threshold above) for sub-allocation.
      uint64_t reserved = 0;
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
      const char *env = getenv("FTT_POOL_RESERVE_MB");
      const size_t want = (size_t)(env ? atoll(env) : 4096) << 20;
      if (want > reserved) {
        void *blk = nullptr;
        if (cudaMallocAsync(&blk, want - reserved, ctx->stream) == cudaSuccess) {
          cudaFreeAsync(blk, ctx->stream);
          cudaStreamSynchronize(ctx->stream);
        } else {
          cudaGetLastError();
        }
      }
    }
  }
  cudaError_t e = cudaMallocHost(&ctx->pinned, 65536);
  if (e == cudaSuccess) memset(ctx->pinned, 0, 65536);
  if (e == cudaSuccess) e = cudaMallocHost((void **)&ctx->ring, kRingBytes);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ring_ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMalloc((void **)&ctx->sticky, 64);
  if (e == cudaSuccess) e = cudaMemset(ctx->sticky, 0, 64);
  if (e == cudaSuccess) e = cudaMalloc((void **)&ctx->tile_cnt, sizeof(unsigned) * (kTileCnt + 64));
  if (e == cudaSuccess) e = cudaMemset(ctx->tile_cnt, 0, sizeof(unsigned) * (kTileCnt + 64));
  if (e != cudaSuccess) {
    if (ctx->tile_cnt) cudaFree(ctx->tile_cnt);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->ring) cudaFreeHost(ctx->ring);
    if (ctx->ring_ev) cudaEventDestroy(ctx->ring_ev);
    if (ctx->sticky) cudaFree(ctx->sticky);
    delete ctx;
    set_error("context buffers: %s", cudaGetErrorString(e));
    return FTT_ERR_CUDA;
  }
  *ctx_out = ctx;
  return FTT_OK;
}

int ftt_destroy(ftt_ctx *ctx) {
  if (!ctx) return FTT_OK;
  cudaSetDevice(ctx->device);
  svd_state_free(ctx);
  for (auto &p : ctx->owned) cudaFreeAsync(p.first, ctx->stream);
  ctx->owned.clear();
  if (ctx->arena.base) cudaFreeAsync(ctx->arena.base, ctx->stream);
  if (ctx->zflags) cudaFreeAsync(ctx->zflags, ctx->stream);
  if (ctx->cp_status) cudaFreeAsync(ctx->cp_status, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->ring) cudaFreeHost(ctx->ring);
  if (ctx->ring_ev) cudaEventDestroy(ctx->ring_ev);
  if (ctx->sticky) cudaFree(ctx->sticky);
  if (ctx->tile_cnt) cudaFree(ctx->tile_cnt);
  delete ctx;
  return FTT_OK;
}

int ftt_set_stream(ftt_ctx *ctx, void *stream) {
  if (!ctx) return FTT_ERR_INVALID;
  if (static_cast<cudaStream_t>(stream) == ctx->stream) return FTT_OK;
  // staged copies and deferred flags of the old stream must land first
  FTT_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->stream = static_cast<cudaStream_t>(stream);
  return FTT_OK;
}

int ftt_set_deferred_checks(ftt_ctx *ctx, int32_t on) {
  if (!ctx) return FTT_ERR_INVALID;
  ctx->defer_checks = on != 0;
  return FTT_OK;
}

int ftt_take_status(ftt_ctx *ctx, int32_t *flags_out) {
  if (!ctx || !flags_out) return FTT_ERR_INVALID;
  int h = 0;
  FTT_CHECK(copy_to_host(ctx, &h, ctx->sticky, sizeof(int)));
  FTT_CUDA(cudaMemsetAsync(ctx->sticky, 0, sizeof(int), ctx->stream));
  *flags_out = h;
  return FTT_OK;
}

int ftt_sync_stats(const ftt_ctx *ctx, int64_t *syncs_out, double *wait_ms_out) {
  if (!ctx) return FTT_ERR_INVALID;
  if (syncs_out) *syncs_out = ctx->syncs;
  if (wait_ms_out) *wait_ms_out = ctx->sync_wait_ms;
  return FTT_OK;
}

int64_t ftt_kernel_launches(const ftt_ctx *ctx) { return ctx ? ctx->launches : 0; }

int ftt_profile_enable(ftt_ctx *ctx, int enable) {
  if (!ctx) return FTT_ERR_INVALID;
  FTT_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->prof = enable != 0;
  ctx->prof_recs.clear();
  ctx->ev_used = 0;
  return FTT_OK;
}

int ftt_profile_read(ftt_ctx *ctx, int32_t tag, double *ms_out, int64_t *launches_out,
                     double *bytes_out, double *flops_out) {
  if (!ctx || tag < 0 || tag >= PT_COUNT) return FTT_ERR_INVALID;
  FTT_CUDA(cudaStreamSynchronize(ctx->stream));
  double ms = 0.0, bytes = 0.0, flops = 0.0;
  int64_t n = 0;
  for (const ProfRec &r : ctx->prof_recs) {
    if (r.tag != tag) continue;
    float t = 0.f;
    FTT_CUDA(cudaEventElapsedTime(&t, ctx->ev_pool[r.ev_a], ctx->ev_pool[r.ev_b]));
    ms += t;
    bytes += r.bytes;
    flops += r.flops;
    ++n;
  }
  if (ms_out) *ms_out = ms;
  if (launches_out) *launches_out = n;
  if (bytes_out) *bytes_out = bytes;
  if (flops_out) *flops_out = flops;
  return FTT_OK;
}

int ftt_set_lin_chunks(ftt_ctx *ctx, int32_t nchunks, const int64_t *ends, void *const *events) {
  if (!ctx || nchunks < 0 || nchunks > 8 || (nchunks && (!ends || !events))) {
    ftt::set_error("ftt_set_lin_chunks: invalid arguments");
    return FTT_ERR_INVALID;
  }
  ctx->lin_nchunks = nchunks;
  for (int j = 0; j < nchunks; ++j) {
    if (!events[j] || ends[j] < (j ? ends[j - 1] : 0)) {
      ctx->lin_nchunks = 0;
      ftt::set_error("ftt_set_lin_chunks: chunk ends must ascend, events must be set");
      return FTT_ERR_INVALID;
    }
    ctx->lin_ends[j] = ends[j];
    ctx->lin_events[j] = (cudaEvent_t)events[j];
  }
  return FTT_OK;
}

}  // extern "C"
