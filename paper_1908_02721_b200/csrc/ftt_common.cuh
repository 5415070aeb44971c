// Shared internals of libfasttt_b200: context, workspace arena, errors.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/fasttt_b200.h"

namespace ftt {

constexpr int kNumSMs = 148;  // B200
constexpr int kTileCnt = 65536;  // split-K tile counters per context (+64 reduction counters)

void set_error(const char *fmt, ...);

struct SvdState;  // ftt_svd.cu

// Kernel classes for the live roofline measurement (ftt_profile_*).
enum ProfTag {
  PT_SORT = 0,     // onesweep radix passes
  PT_HIST = 1,     // key build + digit histograms
  PT_SEGMENT = 2,  // fiber segmentation / compaction
  PT_SWEEP = 3,    // deparallelisation sweep kernels
  PT_SCATTER = 4,  // pivot-core and carry scatters
  PT_GEMM = 5,     // DMMA GEMM
  PT_QR_PANEL = 6, // cooperative Householder panel
  PT_JACOBI = 7,   // block Jacobi step
  PT_ENTRIES = 8,  // tt_entries
  PT_COUNT = 9
};

struct ProfRec {
  int ev_a, ev_b;
  int tag;
  double bytes, flops;
};

// Grow-only device arena.  Every API call resets it; allocations are
// 256-byte aligned bumps.  Growth frees the old block stream-ordered and
// allocates a larger one (so pointers from before a growth in the same call
// are invalid -- callers reserve the total up front with `reserve`).
struct Arena {
  char *base = nullptr;
  size_t cap = 0;
  size_t used = 0;
};

}  // namespace ftt

struct ftt_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  ftt::Arena arena;
  // persistent, independently sized buffers (SVD factors etc.)
  std::vector<std::pair<void *, size_t>> owned;
  ftt::SvdState *svd = nullptr;
  int64_t launches = 0;
  int num_sms = ftt::kNumSMs;
  void *pinned = nullptr;  // small pinned host scratch (64 KiB)
  unsigned post_seq = 0;   // sequence word of the last k_post (copy_to_host)
  // pinned ring for stream-ordered host->device staging without a sync
  // (stage_to_device); one event fences the latest staged copy
  char *ring = nullptr;
  size_t ring_off = 0;
  cudaEvent_t ring_ev = nullptr;
  // deferred status checks: narrow-QR non-finite flags OR into `sticky`
  // (device int) instead of a host round trip per call (ftt_take_status)
  bool defer_checks = false;
  // ||A||_F^2 of the next low-rank operand when the caller knows it (the
  // sweep driver: a scattered carry keeps the norm of S V^T); consumed and
  // cleared by the next ftt_svd_lowrank* call
  double fro2_hint = 0.0;
  // the rank the next low-rank operand is expected to have (the previous
  // step's, set by the sweep driver): the sketch's numerical rank is then
  // read back with the singular values instead of in its own round trip and
  // the step redone if it differs (which also clears spec_ok for the sweep)
  int64_t rank_hint = 0;
  bool spec_ok = true;
  // `lin` still arriving from the host in chunks (ftt_set_lin_chunks): chunk
  // j covers lin[0 .. lin_ends[j]) once lin_events[j] has fired.  Consumed by
  // the next call that reads lin: select_p's forward counts start on the
  // chunks present, everything else waits for the last event.
  // the values' host -> device copy still in flight (ftt_fasttt_lin): waited
  // for by the first kernel that reads them (the fiber emit), so that the
  // key sort, which reads only lin, overlaps the transfer
  cudaEvent_t values_event = nullptr;
  int lin_nchunks = 0;
  int64_t lin_ends[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaEvent_t lin_events[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  // host round trips (copy_to_host) and the host time spent blocked in them
  int64_t syncs = 0;
  double sync_wait_ms = 0.0;
  int *sticky = nullptr;
  // grow-only flag array kept all-zero between uses (the deparallelisation
  // sweeps mark, rank and unmark only the rows they touch)
  uint32_t *zflags = nullptr;
  size_t zflags_cap = 0;
  // split-K tile arrival counters (zero between products; ftt_gemm.cu)
  unsigned *tile_cnt = nullptr;
  // single-pass compaction: per-tile look-back status words tagged with a
  // per-call epoch (never cleared), followed by the tile ticket and the
  // exit counter (reset by the last CTA of each launch)
  uint64_t *cp_status = nullptr;
  size_t cp_status_cap = 0;
  uint32_t cp_epoch = 0;
  // live per-class kernel timing (off by default)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  int ev_used = 0;
  std::vector<ftt::ProfRec> prof_recs;
};

namespace ftt {

#define FTT_CUDA(expr)                                                      \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) {                                                \
      ::ftt::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,          \
                       cudaGetErrorString(_e));                             \
      return _e == cudaErrorMemoryAllocation ? FTT_ERR_OOM : FTT_ERR_CUDA;  \
    }                                                                       \
  } while (0)

#define FTT_CHECK(expr)            \
  do {                             \
    int _s = (expr);               \
    if (_s != FTT_OK) return _s;   \
  } while (0)

#define FTT_LAUNCHED(ctx)                                                  \
  do {                                                                     \
    (ctx)->launches++;                                                     \
    cudaError_t _e = cudaGetLastError();                                   \
    if (_e != cudaSuccess) {                                               \
      ::ftt::set_error("%s:%d launch: %s", __FILE__, __LINE__,             \
                       cudaGetErrorString(_e));                            \
      return FTT_ERR_CUDA;                                                 \
    }                                                                      \
  } while (0)

// Profiling: prof_begin records an event before a launch (returns -1 when
// profiling is off); prof_end records the closing event and the launch's
// algorithmic bytes / flops under `tag`.
int prof_begin(ftt_ctx *ctx);
void prof_end(ftt_ctx *ctx, int begin, int tag, double bytes, double flops);

// Reserve at least `bytes` of arena for this call (must be called before
// taking pointers).  Resets `used`.
int arena_reserve(ftt_ctx *ctx, size_t bytes);
// Bump-allocate from the reserved arena (fails if the reservation is short).
void *arena_take(ftt_ctx *ctx, size_t bytes);

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

template <class T>
inline T *take(ftt_ctx *ctx, size_t count) {
  return static_cast<T *>(arena_take(ctx, align_up(count * sizeof(T))));
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int grid_for(int64_t n, int threads, int per_thread = 1, int max_blocks = 148 * 16) {
  int64_t b = ceil_div(n, (int64_t)threads * per_thread);
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

// Synchronous device->host copy of a few scalars through pinned scratch.
int copy_to_host(ftt_ctx *ctx, void *host, const void *dev, size_t bytes);
int copy_to_device(ftt_ctx *ctx, void *dev, const void *host, size_t bytes);
// Stream-ordered host->device copy through the pinned ring: returns without
// waiting (the host buffer may be reused at once).  Falls back to a
// synchronous copy for transfers larger than the ring.
int stage_to_device(ftt_ctx *ctx, void *dev, const void *host, size_t bytes);
constexpr size_t kRingBytes = 1 << 20;

// The context's zeroed flag array with at least n entries (grown and
// cleared once; callers must leave it all-zero).
int zero_flags(ftt_ctx *ctx, size_t n, uint32_t **out);
// Look-back status for a single-pass compaction over `ntiles` tiles: the
// status words, the ticket pair and this call's epoch (ftt_index.cu).
int compact_status(ftt_ctx *ctx, size_t ntiles, uint64_t **status, unsigned **ticket,
                   uint32_t *epoch);

// Make the stream wait for every pending lin chunk (and forget them).
int lin_chunks_wait_all(ftt_ctx *ctx);

// Persistent device buffer owned by the context (freed on destroy).
int owned_alloc(ftt_ctx *ctx, void **p, size_t bytes);
void owned_free(ftt_ctx *ctx, void *p);

// ----- primitives shared across translation units (ftt_index.cu)
// LSD radix sort of 64-bit keys with optional 32-bit payload over bits
// [0, end_bit).  Result lands in keys_out/vals_out.  Scratch from the arena
// (reserved by the caller with radix_sort_scratch_bytes).
size_t radix_sort_scratch_bytes(int64_t n, bool with_vals);
int radix_sort(ftt_ctx *ctx, const uint64_t *keys_in, const uint32_t *vals_in,
               uint64_t *keys_out, uint32_t *vals_out, int64_t n, int end_bit);

// Deterministic sum of squares (partial must hold kSumSqBlocks + 1 doubles).
constexpr int kSumSqBlocks = 148 * 8;
int sum_squares(ftt_ctx *ctx, int64_t n, const double *x, double *partial, double *out_host);
int sum_squares_dev(ftt_ctx *ctx, int64_t n, const double *x, double *partial, double *out_dev);
// x . y into a device scalar (same deterministic reduction; partial as above)
int dot_dev(ftt_ctx *ctx, int64_t n, const double *x, const double *y, double *partial,
            double *out_dev);

// Exclusive scan of int64 block counts (small arrays, single block).
int scan_block_counts(ftt_ctx *ctx, int64_t *counts, int64_t nblocks, int64_t *total_dev);

}  // namespace ftt
