// Index path of FastTT on B200: radix sort of linearised COO keys, fiber
// segmentation, per-pivot fiber counts, deparallelisation sweeps and the
// pivot-core scatter.  All integer work is bit-exact with the reference
// (tensor.py:374-403, fasttt.py:148-211, 256-259, 537-541).
//
// Design:
//  * keys: one 64-bit mixed-radix key per nonzero, lin(fixed)*n_p + i_p
//    (< prod(dims) < 2^63, check_shape tensor.py:62-66).  Sorting it is the
//    reference's lexsort (pivot coordinate fastest, tensor.py:387-389).
//  * sort: LSD "onesweep" radix sort -- one fused key-build + all-pass
//    histogram kernel, then one kernel per 8-bit digit that ranks a 4096-key
//    tile with warp match.any, finds its global offset by decoupled
//    look-back over per-tile digit counts, stages the tile in shared memory
//    in digit order and writes runs coalesced.  Passes whose digit is
//    constant over all keys are skipped (decided from the histogram).
//  * segment / compaction: warp-striped ballot scans, 4096 items per block,
//    3 phases (count, scan block counts, emit) -- ascending order preserved.
#include <cooperative_groups.h>

#include "ftt_common.cuh"

namespace ftt {
namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 4096 keys
constexpr int RS_MIN_TILE = RS_TILE;            // status sizing
constexpr int RADIX = 256;
constexpr uint32_t FLAG_AGG = 1u << 30;
constexpr uint32_t FLAG_INC = 2u << 30;
constexpr uint32_t VAL_MASK = (1u << 30) - 1;

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

struct KeySpec {
  // key = sum_k coord[k] * mult[k]  (mixed radix, C order over the modes
  // in key order).  mult[pivot] = 1 for fiber keys, 0 for count keys where
  // the pivot is dropped.
  int32_t d;
  int64_t mult[32];
};

// Radix digit of a key for pass `shift` (bits [shift, shift + 8) of the key
// itself: the ordinary LSD sort).
struct DigitShift {
  int shift;
  __device__ __forceinline__ uint32_t operator()(uint64_t k) const {
    return (uint32_t)((k >> shift) & 255);
  }
};

// Fused: build one key per nonzero from coords + per-block digit
// histograms of every pass.  Writes keys and the identity payload.
__global__ void __launch_bounds__(256) k_keys_hist(const int64_t *__restrict__ coords, int64_t n,
                                                   KeySpec spec, int num_passes,
                                                   uint64_t *__restrict__ keys,
                                                   uint32_t *__restrict__ idx,
                                                   uint32_t *__restrict__ ghist) {
  __shared__ uint32_t sh[8][RADIX];
  for (int i = threadIdx.x; i < 8 * RADIX; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const int d = spec.d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t *c = coords + i * d;
    uint64_t key = 0;
    for (int k = 0; k < d; ++k) key += (uint64_t)c[k] * (uint64_t)spec.mult[k];
    keys[i] = key;
    if (idx) idx[i] = (uint32_t)i;
    for (int p = 0; p < num_passes; ++p) atomicAdd(&sh[p][(key >> (8 * p)) & 255], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < num_passes * RADIX; i += blockDim.x) {
    uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(&ghist[i], v);
  }
}

// Histogram of already-built keys (for sorts whose keys come from elsewhere).
__global__ void __launch_bounds__(256) k_hist(const uint64_t *__restrict__ keys, int64_t n,
                                              int num_passes, uint32_t *__restrict__ ghist,
                                              uint32_t *__restrict__ idx) {
  __shared__ uint32_t sh[8][RADIX];
  for (int i = threadIdx.x; i < 8 * RADIX; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t key = keys[i];
    if (idx) idx[i] = (uint32_t)i;
    for (int p = 0; p < num_passes; ++p) atomicAdd(&sh[p][(key >> (8 * p)) & 255], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < num_passes * RADIX; i += blockDim.x) {
    uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(&ghist[i], v);
  }
}

// Exclusive scan of each pass histogram (one block of 256 threads per pass).
__global__ void k_hist_scan(uint32_t *ghist) {
  __shared__ uint32_t s[RADIX];
  uint32_t *h = ghist + blockIdx.x * RADIX;
  int t = threadIdx.x;
  s[t] = h[t];
  __syncthreads();
  for (int off = 1; off < RADIX; off <<= 1) {
    uint32_t v = t >= off ? s[t - off] : 0;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  h[t] = s[t] - h[t];  // exclusive
}

template <bool HAS_VALS, int ITEMS = RS_ITEMS, class DG = DigitShift>
__global__ void __launch_bounds__(RS_THREADS) k_onesweep(
    const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint64_t *__restrict__ kout,
    uint32_t *__restrict__ vout, int64_t n, DG dgf, const uint32_t *__restrict__ digit_start,
    uint32_t *__restrict__ status, uint32_t *__restrict__ tile_counter) {
  __shared__ uint32_t s_warp[RS_WARPS][RADIX];
  __shared__ uint32_t s_excl[RADIX];
  __shared__ uint32_t s_gbase[RADIX];
  __shared__ uint32_t s_wsum[RS_WARPS];
  __shared__ uint32_t s_tile;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  uint64_t *s_keys = reinterpret_cast<uint64_t *>(s_dyn);           // (RS_THREADS * ITEMS) keys
  uint32_t *s_vals = reinterpret_cast<uint32_t *>(s_dyn + 8 * (RS_THREADS * ITEMS));  // (RS_THREADS * ITEMS) payloads

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < RS_WARPS * RADIX; i += RS_THREADS) (&s_warp[0][0])[i] = 0;
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * (RS_THREADS * ITEMS);
  const int64_t wbase = base + warp * (32 * ITEMS);

  uint64_t k[ITEMS];
  uint32_t v[ITEMS];
  uint32_t rank[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    int64_t idx = wbase + i * 32 + lane;
    if (idx < n) {
      k[i] = kin[idx];
      if (HAS_VALS) v[i] = vin[idx];
    } else {
      k[i] = 0;
      if (HAS_VALS) v[i] = 0;
    }
  }
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    int64_t idx = wbase + i * 32 + lane;
    uint32_t dg = idx < n ? dgf(k[i]) : 256u;
    uint32_t peers = __match_any_sync(0xffffffffu, dg);
    int leader = __ffs(peers) - 1;
    uint32_t b = 0;
    if (dg < 256 && lane == leader) {
      b = s_warp[warp][dg];
      s_warp[warp][dg] = b + __popc(peers);
    }
    b = __shfl_sync(0xffffffffu, b, leader);
    rank[i] = b + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive offsets over warps, tile total
  const int dgt = tid;  // RS_THREADS == RADIX
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < RS_WARPS; ++w) {
    uint32_t c = s_warp[w][dgt];
    s_warp[w][dgt] = run;
    run += c;
  }
  const uint32_t total = run;
  // decoupled look-back for this digit
  uint32_t *st = status + tile * RADIX + dgt;
  uint32_t excl = 0;
  if (tile == 0) {
    st_relaxed(st, FLAG_INC | total);
  } else {
    st_relaxed(st, FLAG_AGG | total);
    int64_t j = tile - 1;
    while (true) {
      uint32_t s;
      do {
        s = ld_relaxed(status + j * RADIX + dgt);
      } while ((s & ~VAL_MASK) == 0);
      excl += s & VAL_MASK;
      if ((s & ~VAL_MASK) == FLAG_INC) break;
      --j;
    }
    st_relaxed(st, FLAG_INC | (excl + total));
  }
  s_gbase[dgt] = digit_start[dgt] + excl;
  // block exclusive scan of tile totals over digits -> local staging offsets
  uint32_t x = total;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) s_wsum[warp] = x;
  __syncthreads();
  uint32_t wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
  s_excl[dgt] = wpre + x - total;
  __syncthreads();
  // stage in digit order
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    int64_t idx = wbase + i * 32 + lane;
    if (idx < n) {
      uint32_t dg = dgf(k[i]);
      uint32_t pos = s_excl[dg] + s_warp[warp][dg] + rank[i];
      s_keys[pos] = k[i];
      if (HAS_VALS) s_vals[pos] = v[i];
    }
  }
  __syncthreads();
  const int tile_n = (int)min((int64_t)(RS_THREADS * ITEMS), n - base);
  for (int j = tid; j < tile_n; j += RS_THREADS) {
    uint64_t key = s_keys[j];
    uint32_t dg = dgf(key);
    uint32_t out = s_gbase[dg] + (j - s_excl[dg]);
    kout[out] = key;
    if (HAS_VALS) vout[out] = s_vals[j];
  }
}

// ---- onesweep pass, persistent CTAs with TMA tile prefetch ---------------
// The same pass as k_onesweep (stable 8-bit LSD digit pass: warp match.any
// ranking, decoupled look-back, digit-ordered staging, coalesced runs) but
// each CTA loops over tiles claimed from the tile counter, and as soon as
// the current tile sits in registers the NEXT claimed tile is copied
// global -> shared by the bulk-copy engine (cp.async.bulk, one elected
// thread, completion on an mbarrier), so its HBM latency overlaps this
// tile's ranking, look-back and scatter.  A tile's predecessors are always
// some CTA's current tile or already finished, so the look-back cannot
// deadlock on a prefetched tile.  Tiles whose bytes are not 16-byte
// multiples (the last one) are read with ordinary loads.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

template <bool HAS_VALS, class DG>
__global__ void __launch_bounds__(RS_THREADS, HAS_VALS ? 2 : 3) k_onesweep_tma(
    const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint64_t *__restrict__ kout,
    uint32_t *__restrict__ vout, int64_t n, DG dgf, const uint32_t *__restrict__ digit_start,
    uint32_t *__restrict__ status, uint32_t *__restrict__ tile_counter, int64_t ntiles) {
  constexpr int ITEMS = RS_ITEMS, TILE = RS_TILE;
  __shared__ uint32_t s_warp[RS_WARPS][RADIX];
  __shared__ uint32_t s_excl[RADIX];
  __shared__ uint32_t s_gbase[RADIX];
  __shared__ uint32_t s_wsum[RS_WARPS];
  __shared__ int64_t s_next;
  __shared__ __align__(8) uint64_t s_bar;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  uint64_t *s_keys = reinterpret_cast<uint64_t *>(s_dyn);               // staging keys
  uint32_t *s_vals = reinterpret_cast<uint32_t *>(s_dyn + 8 * TILE);    // staging payloads
  // prefetch buffer after the staging one (keys only: 8 + 8 bytes per key)
  uint64_t *l_keys = reinterpret_cast<uint64_t *>(s_dyn + (HAS_VALS ? 12 : 8) * TILE);
  uint32_t *l_vals = reinterpret_cast<uint32_t *>(s_dyn + 20 * TILE);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt = lanemask_lt();
  auto full_tile = [&](int64_t t) { return (t + 1) * TILE <= n; };
  // claim + prefetch (thread 0); returns the claimed tile via s_next
  auto claim_and_prefetch = [&]() {
    const int64_t t = atomicAdd(tile_counter, 1u);
    s_next = t;
    if (t < ntiles && full_tile(t)) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const unsigned kb = 8u * TILE, vb = HAS_VALS ? 4u * TILE : 0u;
      mbar_expect_tx(&s_bar, kb + vb);
      bulk_g2s(l_keys, kin + t * TILE, kb, &s_bar);
      if (HAS_VALS) bulk_g2s(l_vals, vin + t * TILE, vb, &s_bar);
    }
  };
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    claim_and_prefetch();
  }
  __syncthreads();
  unsigned phase = 0;
  int64_t tile = s_next;
  while (tile < ntiles) {
    for (int i = tid; i < RS_WARPS * RADIX; i += RS_THREADS) (&s_warp[0][0])[i] = 0;
    const int64_t base = tile * TILE;
    const int64_t wbase = base + warp * (32 * ITEMS);
    const int woff = warp * (32 * ITEMS);
    uint64_t k[ITEMS];
    uint32_t v[ITEMS];
    uint32_t rank[ITEMS];
    const bool bulk = full_tile(tile);
    if (bulk) {
      mbar_wait(&s_bar, phase);
      phase ^= 1u;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        k[i] = l_keys[woff + i * 32 + lane];
        if (HAS_VALS) v[i] = l_vals[woff + i * 32 + lane];
      }
    } else {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int64_t idx = wbase + i * 32 + lane;
        k[i] = idx < n ? kin[idx] : 0;
        if (HAS_VALS) v[i] = idx < n ? vin[idx] : 0;
      }
    }
    __syncthreads();  // prefetch buffer consumed, counters cleared
    if (tid == 0) claim_and_prefetch();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int64_t idx = wbase + i * 32 + lane;
      const uint32_t dg = idx < n ? dgf(k[i]) : 256u;
      const uint32_t peers = __match_any_sync(0xffffffffu, dg);
      const int leader = __ffs(peers) - 1;
      uint32_t b = 0;
      if (dg < 256 && lane == leader) {
        b = s_warp[warp][dg];
        s_warp[warp][dg] = b + __popc(peers);
      }
      b = __shfl_sync(0xffffffffu, b, leader);
      rank[i] = b + __popc(peers & lt);
      __syncwarp();
    }
    __syncthreads();
    const int dgt = tid;  // RS_THREADS == RADIX
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
      const uint32_t c = s_warp[w][dgt];
      s_warp[w][dgt] = run;
      run += c;
    }
    const uint32_t total = run;
    uint32_t *st = status + tile * RADIX + dgt;
    uint32_t excl = 0;
    if (tile == 0) {
      st_relaxed(st, FLAG_INC | total);
    } else {
      st_relaxed(st, FLAG_AGG | total);
      int64_t j = tile - 1;
      while (true) {
        uint32_t sv;
        do {
          sv = ld_relaxed(status + j * RADIX + dgt);
        } while ((sv & ~VAL_MASK) == 0);
        excl += sv & VAL_MASK;
        if ((sv & ~VAL_MASK) == FLAG_INC) break;
        --j;
      }
      st_relaxed(st, FLAG_INC | (excl + total));
    }
    s_gbase[dgt] = digit_start[dgt] + excl;
    uint32_t x = total;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    uint32_t wpre = 0;
    for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
    s_excl[dgt] = wpre + x - total;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int64_t idx = wbase + i * 32 + lane;
      if (idx < n) {
        const uint32_t dg = dgf(k[i]);
        const uint32_t pos = s_excl[dg] + s_warp[warp][dg] + rank[i];
        s_keys[pos] = k[i];
        if (HAS_VALS) s_vals[pos] = v[i];
      }
    }
    __syncthreads();
    const int tile_n = (int)min((int64_t)TILE, n - base);
    for (int j = tid; j < tile_n; j += RS_THREADS) {
      const uint64_t key = s_keys[j];
      const uint32_t dg = dgf(key);
      const uint32_t out = s_gbase[dg] + (j - s_excl[dg]);
      kout[out] = key;
      if (HAS_VALS) vout[out] = s_vals[j];
    }
    __syncthreads();  // staging reused by the next tile; s_next published
    tile = s_next;
  }
}

// ---------------------------------------------------------- compaction
// Warp-striped blocks of COMPACT_TILE items.  Pred: bool(int64 i).
constexpr int CP_THREADS = 256;
constexpr int CP_ITEMS = 16;
constexpr int CP_TILE = CP_THREADS * CP_ITEMS;

// Dynamic length: n = min(nmax, *n_dev * mult) when n_dev is given (a count
// produced on the device by an earlier kernel; grids are sized for nmax and
// blocks past n exit).
__device__ __forceinline__ int64_t dyn_n(int64_t nmax, const int64_t *n_dev, int64_t mult) {
  return n_dev ? min(nmax, *n_dev * mult) : nmax;
}

__global__ void k_scan_counts(int64_t *counts, int64_t nb, int64_t *total,
                              const int64_t *n_dev = nullptr, int64_t mult = 1) {
  // single block, 1024 threads, chunked exclusive scan
  if (n_dev) nb = min(nb, (*n_dev * mult + CP_TILE - 1) / CP_TILE);
  __shared__ int64_t s[1024];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += 1024) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < nb ? counts[i] : 0;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      int64_t y = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
      __syncthreads();
      s[threadIdx.x] += y;
      __syncthreads();
    }
    if (i < nb) counts[i] = carry + s[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += s[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

// Single-pass compaction: each CTA claims tiles in order from a ticket,
// ranks its flagged items with warp ballots, publishes the tile total
// (AGG), finds its exclusive prefix by a warp-wide decoupled look-back over
// the 32 nearest predecessors at a time (the nearest INC ends it), publishes
// the inclusive prefix (INC) and emits.  Status words carry this call's
// epoch, so the array is never cleared between calls; the ticket is reset by
// the last CTA to leave.  One launch instead of count + scan + emit.
// Status word: epoch << 34 | flag << 32 | value (counts < 2^32).
constexpr uint64_t CPS_AGG = 1ull, CPS_INC = 2ull;

__device__ __forceinline__ uint64_t ld_relaxed64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <class Pred, class Emit>
__global__ void __launch_bounds__(CP_THREADS) k_compact1(int64_t nmax, Pred pred, Emit emit,
                                                         uint64_t *__restrict__ status,
                                                         unsigned *__restrict__ ticket,
                                                         uint32_t epoch, int64_t *total,
                                                         const int64_t *n_dev, int64_t mult) {
  const int64_t n = dyn_n(nmax, n_dev, mult);
  const int64_t ntile = (n + CP_TILE - 1) / CP_TILE;
  __shared__ int s_w[CP_THREADS / 32];
  __shared__ int64_t s_tile;
  __shared__ uint32_t s_excl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  const uint64_t tag = (uint64_t)epoch << 34;
  if (ntile == 0 && blockIdx.x == 0 && threadIdx.x == 0 && total) *total = 0;
  while (true) {
    if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntile) break;
    const int64_t wbase = tile * CP_TILE + warp * (32 * CP_ITEMS);
    uint32_t balls[CP_ITEMS];
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < CP_ITEMS; ++j) {
      const int64_t i = wbase + j * 32 + lane;
      const bool f = i < n && pred(i);
      balls[j] = __ballot_sync(0xffffffffu, f);
      cnt += __popc(balls[j]);
    }
    if (lane == 0) s_w[warp] = cnt;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < CP_THREADS / 32; ++w) {
      const uint32_t c = (uint32_t)s_w[w];
      wpre += w < warp ? c : 0u;
      tot += c;
    }
    if (warp == 0) {
      uint32_t excl = 0;
      if (tile == 0) {
        if (lane == 0) st_relaxed64(status, tag | (CPS_INC << 32) | tot);
      } else {
        if (lane == 0) st_relaxed64(status + tile, tag | (CPS_AGG << 32) | tot);
        int64_t j = tile - 1 - lane;  // lane 0 = nearest predecessor
        while (true) {
          const uint64_t sw = j >= 0 ? ld_relaxed64(status + j) : (tag | (CPS_INC << 32));
          const bool valid = (sw >> 34) == epoch && ((sw >> 32) & 3u) != 0;
          if (!__all_sync(0xffffffffu, valid)) continue;
          const unsigned inc = __ballot_sync(0xffffffffu, ((sw >> 32) & 3u) == CPS_INC);
          const int stop = inc ? __ffs(inc) - 1 : 31;
          uint32_t v = lane <= stop ? (uint32_t)sw : 0u;
#pragma unroll
          for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          excl += v;
          if (inc) break;
          j -= 32;
        }
        if (lane == 0) st_relaxed64(status + tile, tag | (CPS_INC << 32) | (uint32_t)(excl + tot));
      }
      if (lane == 0) {
        s_excl = excl;
        if (tile == ntile - 1 && total) *total = (int64_t)excl + tot;
      }
    }
    __syncthreads();
    int64_t run = (int64_t)s_excl + wpre;
    if constexpr (Emit::kTwoPhase) {
      constexpr int CP_BATCH = 8;  // items whose gathers are in flight together (16: spills, 284 us)
#pragma unroll
      for (int j0 = 0; j0 < CP_ITEMS; j0 += CP_BATCH) {
        typename Emit::Item it[CP_BATCH];
#pragma unroll
        for (int u = 0; u < CP_BATCH; ++u) {
          const int64_t i = wbase + (j0 + u) * 32 + lane;
          if (i < n) it[u] = emit.load(i);
        }
#pragma unroll
        for (int u = 0; u < CP_BATCH; ++u) {
          const int j = j0 + u;
          const int64_t i = wbase + j * 32 + lane;
          const bool f = (balls[j] >> lane) & 1u;
          if (i < n) emit.store(i, run + __popc(balls[j] & lt), f, it[u]);
          run += __popc(balls[j]);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < CP_ITEMS; ++j) {
        const int64_t i = wbase + j * 32 + lane;
        const bool f = (balls[j] >> lane) & 1u;
        if (i < n) emit(i, run + __popc(balls[j] & lt), f);
        run += __popc(balls[j]);
      }
    }
    __syncthreads();  // s_tile / s_w / s_excl reuse
  }
  if (threadIdx.x == 0) {
    __threadfence();  // this CTA's last ticket claim before its exit count
    if (atomicAdd(ticket + 1, 1u) == gridDim.x - 1) {
      __threadfence();
      ticket[0] = 0;
      ticket[1] = 0;
    }
  }
}

// `tag`/`alg_bytes`: profiling class and algorithmic bytes of the whole
// compaction (predicate reads + emitted outputs).  `block_counts` is unused
// (kept for the callers' scratch layout).  n < 2^31 (every caller).
template <class Pred, class Emit>
int compact(ftt_ctx *ctx, int64_t n, Pred pred, Emit emit, int64_t *block_counts,
            int64_t *total_dev, int tag = PT_SEGMENT, double alg_bytes = 0.0,
            const int64_t *n_dev = nullptr, int64_t mult = 1) {
  (void)block_counts;
  if (n <= 0) return FTT_OK;
  if (n >= ((int64_t)1 << 31)) {
    set_error("compaction length %lld exceeds 2^31", (long long)n);
    return FTT_ERR_INVALID;
  }
  const int64_t nb = ceil_div(n, CP_TILE);
  uint64_t *status = nullptr;
  unsigned *ticket = nullptr;
  uint32_t epoch = 0;
  FTT_CHECK(compact_status(ctx, (size_t)nb, &status, &ticket, &epoch));
  // dynamic lengths: a bounded grid claims the live tiles
  const unsigned grid = (unsigned)std::min<int64_t>(nb, 8 * (int64_t)ctx->num_sms);
  const int pb = tag >= 0 ? prof_begin(ctx) : -1;
  k_compact1<Pred, Emit><<<grid, CP_THREADS, 0, ctx->stream>>>(n, pred, emit, status, ticket,
                                                               epoch, total_dev, n_dev, mult);
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb, tag, alg_bytes, 0.0);
  return FTT_OK;
}

inline size_t compact_scratch_bytes(int64_t n) {
  return align_up(sizeof(int64_t) * (ceil_div(n, CP_TILE) + 1)) + 256;
}

// ------------------------------------------------------------- functors
// Exact division of x < 2^63 by a run-time constant D: floor(x / D) =
// mulhi(x, m) >> sh (Granlund-Montgomery with N = 63; D = 1 -> sh = -1).
// 64-bit integer division is a ~70-instruction software routine on the GPU;
// the segment and sweep kernels divide every element.
struct Div63 {
  uint64_t d, m;
  int sh;
  __device__ __forceinline__ uint64_t quo(uint64_t x) const { return sh < 0 ? x : (__umul64hi(x, m) >> sh); }
};

Div63 make_div63(uint64_t D) {
  Div63 r;
  r.d = D;
  if (D <= 1) {
    r.m = 0;
    r.sh = -1;
    return r;
  }
  int l = 0;
  while (((unsigned __int128)1 << l) < D) ++l;
  const unsigned __int128 num = (unsigned __int128)1 << (63 + l);
  r.m = (uint64_t)(num / D + 1);
  r.sh = l - 1;
  return r;
}

struct AdjDiffPred {  // sorted keys: key/div differs from predecessor
  const uint64_t *k;
  Div63 div;
  __device__ bool operator()(int64_t i) const {
    return i == 0 || div.quo(k[i]) != div.quo(k[i - 1]);
  }
};

struct FiberEmit {
  static constexpr bool kTwoPhase = false;
  const uint64_t *k;
  const uint32_t *perm;
  const double *vals_in;
  Div63 np;
  int64_t *fixed_lin, *indptr, *fiber_of, *pivot_index;
  double *vals_out;
  __device__ void operator()(int64_t i, int64_t r, bool f) const {
    uint64_t key = k[i];
    uint64_t fx = np.quo(key);
    if (f) {
      indptr[r] = i;
      fixed_lin[r] = (int64_t)fx;
    }
    if (fiber_of) fiber_of[i] = f ? r : r - 1;
    pivot_index[i] = (int64_t)(key - fx * np.d);
    vals_out[i] = vals_in[perm[i]];
  }
};

struct FlagPred {
  const uint32_t *present;
  __device__ bool operator()(int64_t i) const { return present[i] != 0; }
};

struct KeptEmit {  // kept[r] = row, present[row] <- rank (overwrites the flag)
  static constexpr bool kTwoPhase = false;
  uint32_t *present;
  int64_t *kept;
  __device__ void operator()(int64_t i, int64_t r, bool f) const {
    if (f) {
      kept[r] = i;
      present[i] = (uint32_t)r;
    }
  }
};

struct UniqEmit {  // sort path: sorted keys with fiber payload
  static constexpr bool kTwoPhase = false;
  const uint64_t *k;
  const uint32_t *perm;
  int64_t *kept, *map_out;
  __device__ void operator()(int64_t i, int64_t r, bool f) const {
    if (f) kept[r] = (int64_t)k[i];
    map_out[perm[i]] = f ? r : r - 1;
  }
};

struct SweepKey {
  int32_t side;
  const int64_t *fixed_lin;
  int64_t stride, nk, r_other;
  const int64_t *map_in;
  Div63 dstride, dnk;
  const int64_t *r_other_dev = nullptr;  // device-resident r_other (batched sweeps)
  __device__ int64_t operator()(int64_t f) const { return with_map(f, map_in ? map_in[f] : 0); }
  // the key with the previous step's map value m given (fused kernels)
  __device__ int64_t with_map(int64_t f, int64_t m) const {
    const uint64_t q = dstride.quo((uint64_t)fixed_lin[f]);
    int64_t ik = (int64_t)(q - dnk.quo(q) * (uint64_t)nk);
    const int64_t ro = r_other_dev ? *r_other_dev : r_other;
    return side == 0 ? m * nk + ik : ik * ro + m;
  }
};

// present[kept[r]] = 0 for r < *count (undo one step's marks / ranks).
__global__ void k_unmark(const int64_t *__restrict__ kept, const int64_t *__restrict__ count,
                         int64_t bound, uint32_t *__restrict__ present) {
  const int64_t n = min(*count, bound);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    present[kept[r]] = 0u;
}

// (Marks test the flag first: the early steps have millions of fibers on a few
// dozen rows, and unconditional stores to the same words serialise in L2 --
// 64 us for a 32-row step against 13 us for a 3 M-row one.  A stale 0 from L1
// only costs a redundant store.)
__global__ void k_sweep_mark(int64_t R, SweepKey key, uint32_t *present) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < R;
       f += (int64_t)gridDim.x * blockDim.x) {
    uint32_t *p = present + key(f);
    if (*p == 0u) *p = 1u;
  }
}

__global__ void k_sweep_gather(int64_t R, SweepKey key, const uint32_t *present, int64_t *map_out) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < R;
       f += (int64_t)gridDim.x * blockDim.x)
    map_out[f] = (int64_t)present[key(f)];
}

// Step s's gather fused with step s+1's mark: map_s[f] = rank of key_s(f),
// then key_{s+1}(f) -- which needs exactly that map value (same side) or
// none (first step of the other side) -- is marked in the other flag array.
// One pass over the fibers per step instead of two.
__global__ void k_sweep_gather_mark(int64_t R, SweepKey key, const uint32_t *present,
                                    int64_t *map_out, SweepKey next, int next_uses_map,
                                    uint32_t *present_next) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < R;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = (int64_t)present[key(f)];
    map_out[f] = m;
    uint32_t *p = present_next + next.with_map(f, next_uses_map ? m : 0);
    if (*p == 0u) *p = 1u;
  }
}

__global__ void k_sweep_keys(int64_t R, SweepKey key, uint64_t *keys) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < R;
       f += (int64_t)gridDim.x * blockDim.x)
    keys[f] = (uint64_t)key(f);
}

__global__ void k_mark_rows(int64_t n, const int64_t *rows, uint32_t *present) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    present[rows[i]] = 1u;
}

__global__ void k_gather_rank(int64_t n, const int64_t *rows, const uint32_t *present, int64_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)present[rows[i]];
}

__global__ void k_copy_keys(int64_t n, const int64_t *in, uint64_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint64_t)in[i];
}

__global__ void k_set_i64(int64_t *p, int64_t v) { *p = v; }

constexpr int HS_MAXP = 32;
constexpr int HS_PASS = 16;  // pivots per launch (first probes held in registers)
// Key with the mode-q digit removed from the C-order linear index:
// (lin / T_q) * S_q + lin % S_q with S_q = prod of the dims after q and
// T_q = n_q S_q (exact magic-number divisions, lin < 2^63).
struct HashSpec {
  int d, np, lg;
  int64_t stride[32];  // C-order strides of the full index
  uint64_t S[HS_MAXP], mS[HS_MAXP], mT[HS_MAXP];
  int shS[HS_MAXP], shT[HS_MAXP];
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t hs_div(uint64_t x, uint64_t m, int sh) {
  return sh < 0 ? x : (__umul64hi(x, m) >> sh);
}
__device__ __forceinline__ uint64_t sm_div(uint64_t x, uint64_t m, int sh) { return hs_div(x, m, sh); }

// Insert the np fixed-tuple keys of every nonzero into np hash sets (empty
// slot = ~0, keys < 2^63); count first insertions per set.  One nonzero per
// thread: the linear index is accumulated straight from the coordinates,
// each pivot's key derived from it, and the first probe of every pivot is
// issued before any result is examined (independent atomics in flight);
// collisions (rare at load factor <= 1/2) then probe linearly.
__global__ void __launch_bounds__(256) k_distinct_hash(const int64_t *__restrict__ coords,
                                                       const uint64_t *__restrict__ lin_in, int64_t n,
                                                       HashSpec hs,
                                                       unsigned long long *__restrict__ tables,
                                                       unsigned long long *__restrict__ counts) {
  const int64_t T = (int64_t)1 << hs.lg;
  const uint64_t mask = (uint64_t)T - 1;
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    uint64_t lin = 0;
    if (i < n) {
      if (lin_in) {
        lin = lin_in[i];
      } else {
        const int64_t *c = coords + i * hs.d;
        for (int k = 0; k < hs.d; ++k) lin += (uint64_t)c[k] * (uint64_t)hs.stride[k];
      }
    }
    unsigned fresh_mask = 0, pending = 0;
    unsigned long long got[HS_PASS];
    auto key_of = [&](int q) -> uint64_t {
      const uint64_t hi = hs_div(lin, hs.mT[q], hs.shT[q]);
      const uint64_t lo = lin - hs_div(lin, hs.mS[q], hs.shS[q]) * hs.S[q];
      return hi * hs.S[q] + lo;
    };
#pragma unroll
    for (int q = 0; q < HS_PASS; ++q) {
      got[q] = 0;
      if (q >= hs.np || i >= n) continue;
      const uint64_t k = key_of(q);
      got[q] = atomicCAS(tables + (int64_t)q * T + (mix64(k) & mask), ~0ull, (unsigned long long)k);
    }
#pragma unroll
    for (int q = 0; q < HS_PASS; ++q) {
      if (q >= hs.np || i >= n) continue;
      if (got[q] == ~0ull) fresh_mask |= 1u << q;
      else if (got[q] != key_of(q)) pending |= 1u << q;
    }
    while (pending) {  // linear probing for the colliding pivots
      const int q = __ffs(pending) - 1;
      pending &= pending - 1;
      unsigned long long *tab = tables + (int64_t)q * T;
      const uint64_t k = key_of(q);
      uint64_t h = mix64(k) & mask;
      while (true) {
        h = (h + 1) & mask;
        const unsigned long long old = atomicCAS(tab + h, ~0ull, (unsigned long long)k);
        if (old == ~0ull) {
          fresh_mask |= 1u << q;
          break;
        }
        if (old == k) break;
      }
    }
    for (int q = 0; q < hs.np; ++q) {
      const unsigned b = __ballot_sync(0xffffffffu, (fresh_mask >> q) & 1u);
      if (lane == 0 && b) atomicAdd(counts + q, (unsigned long long)__popc(b));
    }
  }
}

// ---- partitioned distinct counts (select_p on large inputs) --------------
// Exact number of distinct fixed tuples per pivot p without sorting:
//   lin   = C-order linear index of each nonzero (< 2^63, one pass over COO)
//   key_p = lin with the mode-p digit removed = (lin / T_p) S_p + lin mod S_p
//           (S_p = prod of the dims after p, T_p = n_p S_p; division by
//           run-time constants via exact 64-bit magic multipliers)
//   bucket = top `bits` bits of mix64(key_p): equal keys share a bucket
//   pass 1 per-block bucket histograms, pass 2 scatter into bucket segments,
//   pass 3 one CTA per bucket counts distinct keys in a shared-memory hash
//   set (slot = low bits of the same mix).  Counting is insertion-order
//   independent, so the result is exact and deterministic; a bucket too large
//   for the shared table flags its pivot, which is then counted by sorting.
constexpr int PC_MAXG = 8;
constexpr int PC_TMAX = 8192;  // shared hash-set slots (64 KB)
struct PartSpec {
  int g, bits;
  int64_t chunk;  // nonzeros per block
  uint64_t S[PC_MAXG], mS[PC_MAXG], mT[PC_MAXG];
  int shS[PC_MAXG], shT[PC_MAXG];  // -1: divisor 1
};

__device__ __forceinline__ uint64_t udiv_magic(uint64_t x, uint64_t m, int sh) {
  return sh < 0 ? x : (__umul64hi(x, m) >> sh);
}

__device__ __forceinline__ uint64_t drop_digit(uint64_t lin, const PartSpec &ps, int q) {
  const uint64_t hi = udiv_magic(lin, ps.mT[q], ps.shT[q]);
  const uint64_t lo = lin - udiv_magic(lin, ps.mS[q], ps.shS[q]) * ps.S[q];
  return hi * ps.S[q] + lo;
}

struct LinSpec {
  int d;
  int64_t stride[32];
};

__global__ void __launch_bounds__(256) k_linearize(const int64_t *__restrict__ coords, int64_t n,
                                                   LinSpec ls, uint64_t *__restrict__ lin) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t *c = coords + i * ls.d;
    uint64_t x = 0;
    for (int k = 0; k < ls.d; ++k) x += (uint64_t)c[k] * (uint64_t)ls.stride[k];
    lin[i] = x;
  }
}

// One pass per pivot group: each block histograms its chunk of `lin` per
// (pivot, bucket) in shared memory, reserves that many slots of the bucket's
// fixed-capacity region with one global atomic per non-empty counter, then
// re-reads the chunk (L2-resident) and scatters the keys into its reserved
// runs.  Bucket order inside a region is arbitrary -- the distinct count is
// order independent -- so no global histogram / scan pass is needed.  A
// bucket that outgrows its capacity flags its pivot (sort-path fallback).
__global__ void __launch_bounds__(1024) k_part_scatter(const uint64_t *__restrict__ lin, int64_t n,
                                                       PartSpec ps, int64_t cap,
                                                       unsigned int *__restrict__ fill,
                                                       uint64_t *__restrict__ keys,
                                                       int *__restrict__ flags) {
  extern __shared__ unsigned int cur[];
  const int nbk = 1 << ps.bits, tot = ps.g * nbk;
  for (int e = threadIdx.x; e < tot; e += blockDim.x) cur[e] = 0;
  __syncthreads();
  const int64_t i0 = blockIdx.x * ps.chunk, i1 = min(n, i0 + ps.chunk);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const uint64_t x = lin[i];
#pragma unroll 4
    for (int q = 0; q < ps.g; ++q) {
      const uint32_t b = (uint32_t)(mix64(drop_digit(x, ps, q)) >> (64 - ps.bits));
      atomicAdd(&cur[q * nbk + b], 1u);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    const unsigned int c = cur[e];
    if (c) {
      const unsigned int off = atomicAdd(&fill[e], c);
      if ((int64_t)off + c > cap) flags[e / nbk] = 1;
      cur[e] = off;
    }
  }
  __syncthreads();
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const uint64_t x = lin[i];
#pragma unroll 4
    for (int q = 0; q < ps.g; ++q) {
      const uint64_t key = drop_digit(x, ps, q);
      const uint32_t b = (uint32_t)(mix64(key) >> (64 - ps.bits));
      const int e = q * nbk + b;
      const unsigned int pos = atomicAdd(&cur[e], 1u);
      if (pos < cap) keys[(int64_t)e * cap + pos] = key;
    }
  }
}

// One CTA per (bucket, pivot): distinct keys of the bucket via a shared
// open-addressing set (slot = low bits of the same mix; the bucket fixed its
// top bits).  Counts are exact and independent of the insertion order.
__global__ void __launch_bounds__(256) k_part_count(const uint64_t *__restrict__ keys, int64_t cap,
                                                    const unsigned int *__restrict__ fill, int nbk,
                                                    unsigned long long *__restrict__ counts,
                                                    int *__restrict__ flags) {
  extern __shared__ unsigned long long tab[];
  __shared__ unsigned long long s_cnt;
  const int b = blockIdx.x, q = blockIdx.y;
  const int e = q * nbk + b;
  const int64_t len = fill[e];
  if (len == 0) return;
  if (len > cap) return;  // flagged by the scatter
  int T = 64;
  while (T < 2 * len) T <<= 1;
  if (T > PC_TMAX) {
    if (threadIdx.x == 0) flags[q] = 1;
    return;
  }
  for (int j = threadIdx.x; j < T; j += blockDim.x) tab[j] = ~0ull;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const uint64_t mask = (uint64_t)T - 1;
  const uint64_t *src = keys + (int64_t)e * cap;
  unsigned long long fresh = 0;
  for (int j = threadIdx.x; j < len; j += blockDim.x) {
    const uint64_t key = __ldcs(src + j);
    uint64_t h = mix64(key) & mask;
    while (true) {
      const unsigned long long old = atomicCAS(tab + h, ~0ull, (unsigned long long)key);
      if (old == ~0ull) {
        ++fresh;
        break;
      }
      if (old == key) break;
      h = (h + 1) & mask;
    }
  }
  for (int off = 16; off; off >>= 1) fresh += __shfl_down_sync(0xffffffffu, fresh, off);
  if ((threadIdx.x & 31) == 0 && fresh) atomicAdd(&s_cnt, fresh);
  __syncthreads();
  if (threadIdx.x == 0 && s_cnt) atomicAdd(counts + q, s_cnt);
}

// ---- select_p counts from a sorted order (group-local shared hash) ------
// With the linear keys K = sum_k c_k w_k sorted (C order: the canonical
// input; or the reversed-mode order after one radix sort), the nonzeros of a
// pivot-p fiber share hi = K / T_p (T_p = w_p n_p) and lo = K mod w_p, and
// all nonzeros with the same hi are contiguous.  A CTA takes a group-aligned
// chunk (whole hi-groups, <= GC_CAP entries) and counts distinct dropped
// keys hi w_p + lo in a shared-memory hash set: one streaming read of the
// sorted keys per pivot, no scatter.  A group longer than the cap flags the
// pivot (the other order, then the partition path, count it instead).
constexpr int GC_L = 1024;       // nominal entries per CTA
constexpr int GC_CAP = 2048;     // max entries per chunk (hash load <= 1/2)
constexpr int GC_SLOTS = 4096;
static_assert(8 * GC_CAP + 4 * GC_SLOTS <= 8 * GC_SLOTS, "keys + positions fit the dynamic smem");

// Both linear keys of every nonzero in one read of the COO: C order (lin)
// and the reversed-mode order (rlin).
__global__ void __launch_bounds__(256) k_linearize2(const int64_t *__restrict__ coords, int64_t n,
                                                    LinSpec ls, LinSpec rs,
                                                    uint64_t *__restrict__ lin,
                                                    uint64_t *__restrict__ rlin) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t *c = coords + i * ls.d;
    uint64_t x = 0, y = 0;
    for (int k = 0; k < ls.d; ++k) {
      const uint64_t v = (uint64_t)c[k];
      x += v * (uint64_t)ls.stride[k];
      y += v * (uint64_t)rs.stride[k];
    }
    lin[i] = x;
    rlin[i] = y;
  }
}

// coords[i][k] = digit k of the C-order linear index lin[i] (the inverse of
// linearize, tensor.py:75-100), magic-number divisions by the strides.
struct DelinSpec {
  int d;
  int64_t stride[32];
  uint64_t m[32];
  int sh[32];
};
__global__ void k_delinearize(const int64_t *__restrict__ lin, int64_t n, DelinSpec ds,
                              int64_t *__restrict__ coords) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)lin[i];
    int64_t *c = coords + i * ds.d;
    for (int k = 0; k < ds.d; ++k) {
      const uint64_t q = udiv_magic(x, ds.m[k], ds.sh[k]);
      c[k] = (int64_t)q;
      x -= q * (uint64_t)ds.stride[k];
    }
  }
}

__global__ void k_sorted_check(const uint64_t *__restrict__ k, int64_t n, int *__restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (k[i] <= k[i - 1]) atomicOr(bad, 1);
}

__global__ void __launch_bounds__(256) k_group_count(const uint64_t *__restrict__ K, int64_t n,
                                                     uint64_t S, uint64_t mS, int shS, uint64_t mT,
                                                     int shT, unsigned long long *__restrict__ count,
                                                     int *__restrict__ flag) {
  extern __shared__ unsigned long long tab[];  // GC_SLOTS
  __shared__ int64_t s_start, s_end;
  __shared__ unsigned long long s_cnt;
  const int lane = threadIdx.x & 31;
  const int64_t c0 = (int64_t)blockIdx.x * GC_L;
  auto grp = [&](int64_t i) -> uint64_t { return sm_div(K[i], mT, shT); };
  // first group start >= c0 and >= c0 + L: the CTA tests 256 consecutive
  // positions per round (keys sorted, so grp is monotone) and stops at the
  // first round holding a boundary; no boundary within CAP -> "none"
  __shared__ unsigned s_j[2];
  if (threadIdx.x < 2) s_j[threadIdx.x] = 0xffffffffu;
  __syncthreads();
  // both windows advance together (one dependent load round for the
  // common case of a boundary within the first 256 positions of each)
  bool open0 = c0 < n, open1 = c0 + GC_L < n;
  for (int r = 0; r < GC_CAP / 256 && (open0 || open1); ++r) {
    const int j = r * 256 + (int)threadIdx.x;
    bool st0 = false, st1 = false;
    if (open0) {
      const int64_t i = c0 + j;
      st0 = i <= n && (i == n || i == 0 || grp(i) != grp(i - 1));
    }
    if (open1) {
      const int64_t i = c0 + GC_L + j;
      st1 = i <= n && (i == n || grp(i) != grp(i - 1));
    }
    const unsigned m0 = __reduce_min_sync(0xffffffffu, st0 ? (unsigned)j : 0xffffffffu);
    const unsigned m1 = __reduce_min_sync(0xffffffffu, st1 ? (unsigned)j : 0xffffffffu);
    if (lane == 0 && m0 != 0xffffffffu) atomicMin(&s_j[0], m0);
    if (lane == 0 && m1 != 0xffffffffu) atomicMin(&s_j[1], m1);
    const int any0 = __syncthreads_or(st0);
    const int any1 = __syncthreads_or(st1);
    open0 = open0 && !any0;
    open1 = open1 && !any1;
  }
  if (threadIdx.x == 0) {
    s_start = c0 >= n ? n : (s_j[0] == 0xffffffffu ? INT64_MAX : c0 + s_j[0]);
    s_end = c0 + GC_L >= n ? n : (s_j[1] == 0xffffffffu ? INT64_MAX : c0 + GC_L + s_j[1]);
  }
  __syncthreads();
  const int64_t start = s_start, end = s_end;
  if (start == INT64_MAX) return;  // a long group covers the window; its owner decides
  if (end == INT64_MAX || end - start > GC_CAP) {
    if (threadIdx.x == 0) atomicOr(flag, 1);
    return;
  }
  // the chunk's reduced keys go to shared memory and the hash table holds
  // 32-bit chunk positions (native 32-bit shared CAS; the 64-bit CAS is a
  // spin loop on this part); a probe compares the stored keys
  constexpr int PER = GC_CAP / 256;
  uint64_t *skey = reinterpret_cast<uint64_t *>(tab);        // GC_CAP keys
  unsigned *tab32 = reinterpret_cast<unsigned *>(skey + GC_CAP);  // GC_SLOTS positions
  const int cnt = (int)(end - start);
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = q * 256 + threadIdx.x;
    if (j < cnt) {
      const uint64_t k = __ldg(K + start + j);
      const uint64_t hi = sm_div(k, mT, shT);
      const uint64_t lo = k - sm_div(k, mS, shS) * S;
      skey[j] = hi * S + lo;
    }
  }
  for (int e = threadIdx.x; e < GC_SLOTS / 4; e += blockDim.x)
    reinterpret_cast<uint4 *>(tab32)[e] = make_uint4(~0u, ~0u, ~0u, ~0u);
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  unsigned long long fresh = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = q * 256 + threadIdx.x;
    if (j >= cnt) break;
    const uint64_t key = skey[j];
    uint64_t h = mix64(key) & (GC_SLOTS - 1);
    while (true) {
      const unsigned old = atomicCAS(tab32 + h, ~0u, (unsigned)j);
      if (old == ~0u) {
        ++fresh;
        break;
      }
      if (skey[old] == key) break;
      h = (h + 1) & (GC_SLOTS - 1);
    }
  }
  for (int o = 16; o; o >>= 1) fresh += __shfl_down_sync(0xffffffffu, fresh, o);
  if (lane == 0 && fresh) atomicAdd(&s_cnt, fresh);
  __syncthreads();
  if (threadIdx.x == 0 && s_cnt) atomicAdd(count, s_cnt);
}

__global__ void k_count_changes(const uint64_t *k, int64_t n, unsigned long long *out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += (i == 0 || k[i] != k[i - 1]) ? 1ull : 0ull;
  for (int off = 16; off; off >>= 1) c += __shfl_down_sync(0xffffffffu, c, off);
  __shared__ unsigned long long s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    atomicAdd(out, t);
  }
}

__global__ void k_mode_index(const int64_t *fixed_lin, int64_t R, int64_t stride, int64_t n,
                             int64_t *out) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < R;
       f += (int64_t)gridDim.x * blockDim.x)
    out[f] = (fixed_lin[f] / stride) % n;
}

__global__ void k_pivot_scatter(int64_t nnz, const int64_t *__restrict__ fiber_of,
                                const int64_t *__restrict__ pidx, const double *__restrict__ vals,
                                const int64_t *__restrict__ t_map, const int64_t *__restrict__ s_map,
                                int64_t np, int64_t r_next, double *__restrict__ core,
                                double *__restrict__ partial) {
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t f = fiber_of[e];
    int64_t row = t_map ? t_map[f] : 0;
    int64_t col = s_map ? s_map[f] : 0;
    double v = vals[e];
    core[(row * np + pidx[e]) * r_next + col] = v;
    acc += v * v;
  }
  if (partial) {
    for (int off = 16; off; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
    __shared__ double s[32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
      partial[blockIdx.x] = t;
    }
  }
}

// deterministic final reduction of block partials
__global__ void k_reduce_partials(const double *partial, int nb, double *out) {
  __shared__ double s[1024];
  double a = 0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) a += partial[i];
  s[threadIdx.x] = a;
  __syncthreads();
  for (int off = blockDim.x / 2; off; off >>= 1) {
    if ((int)threadIdx.x < off) s[threadIdx.x] += s[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// Block partials of x.y (x.x when y == nullptr).  With `out` set, the last
// block to finish (arrival counter, reset by it) also sums the partials in
// index order into *out -- one launch instead of two, same result for the
// same grid.
__global__ void __launch_bounds__(256) k_dot_partial(int64_t n, const double *__restrict__ x,
                                                     const double *__restrict__ y, double *partial,
                                                     double *out = nullptr,
                                                     unsigned *counter = nullptr) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc += x[i] * (y ? y[i] : x[i]);
  for (int off = 16; off; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
  __shared__ double s[32];
  __shared__ int s_last;
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    partial[blockIdx.x] = t;
    if (out) {
      __threadfence();
      const unsigned tk = atomicAdd(counter, 1u);
      s_last = tk == gridDim.x - 1;
      if (s_last) *counter = 0u;
    }
  }
  if (!out) return;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  __shared__ double r[256];
  double a = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) a += __ldcg(partial + i);
  r[threadIdx.x] = a;
  __syncthreads();
  for (int off = blockDim.x / 2; off; off >>= 1) {
    if ((int)threadIdx.x < off) r[threadIdx.x] += r[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = r[0];
}

__global__ void k_side_core(int32_t side, const int64_t *kept, int64_t K, int64_t n, int64_t ro,
                            double *core) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < K;
       j += (int64_t)gridDim.x * blockDim.x) {
    int64_t kj = kept[j];
    if (side == 0) {
      // (ro, n, K): [kj / n, kj % n, j] -> ((kj/n)*n + kj%n)*K + j = kj*K + j
      core[kj * K + j] = 1.0;
    } else {
      // (K, n, ro): [j, kj / ro, kj % ro] -> j*(n*ro) + kj
      core[j * (n * ro) + kj] = 1.0;
    }
  }
}

__global__ void k_scatter_cols(int64_t rank, int64_t K, const int64_t *__restrict__ kept,
                               const double *__restrict__ src, int64_t lds, int64_t ncols,
                               double *__restrict__ dst) {
  int64_t total = rank * K;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = t / K, j = t - a * K;
    dst[a * ncols + kept[j]] = src[a * lds + j];
  }
}

__global__ void k_scatter_rows(int64_t K, int64_t rank, const int64_t *__restrict__ kept,
                               const double *__restrict__ src, int64_t lds,
                               double *__restrict__ dst) {
  int64_t total = rank * K;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / rank, c = t - j * rank;
    dst[kept[j] * rank + c] = src[j * lds + c];
  }
}

// ---- tensorize_matrix on the device (ttformat.py:414-433) ------------------
struct FuseSpec {
  int d;
  int64_t rdims[32], cdims[32], stride[32];  // stride: C order over fused dims
};

// fused C-order key of matrix entry (row, col): digits x_i of row over
// row_dims, y_i of col over col_dims, f_i = x_i * c_i + y_i.
__global__ void k_fuse_keys(int64_t nnz, const int64_t *__restrict__ rows,
                            const int64_t *__restrict__ cols, FuseSpec fs,
                            uint64_t *__restrict__ keys, uint32_t *__restrict__ ident,
                            int *__restrict__ bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = rows[e], c = cols[e];
    uint64_t key = 0;
    bool ok = r >= 0 && c >= 0;
    for (int i = fs.d - 1; i >= 0; --i) {
      const int64_t x = r % fs.rdims[i], y = c % fs.cdims[i];
      r /= fs.rdims[i];
      c /= fs.cdims[i];
      key += (uint64_t)(x * fs.cdims[i] + y) * (uint64_t)fs.stride[i];
    }
    if (r != 0 || c != 0) ok = false;  // outside the matrix extents
    if (!ok) atomicOr(bad, 1);
    keys[e] = key;
    ident[e] = (uint32_t)e;
  }
}

// Run of equal keys starting at a head: values summed in input (stable sort)
// order, the scipy tocsr() coalescing; zero sums are dropped like the
// SparseTensor constructor does (tensor.py:147-153).
struct CoalescePred {
  const uint64_t *k;
  const uint32_t *perm;
  const double *v;
  int64_t n;
  __device__ double run_sum(int64_t i) const {
    double s = v[perm[i]];
    for (int64_t j = i + 1; j < n && k[j] == k[i]; ++j) s += v[perm[j]];
    return s;
  }
  __device__ bool operator()(int64_t i) const {
    if (i > 0 && k[i] == k[i - 1]) return false;
    return run_sum(i) != 0.0;
  }
};

struct CoalesceEmit {
  static constexpr bool kTwoPhase = false;
  CoalescePred p;
  FuseSpec fs;
  int64_t *coords;
  double *vals;
  __device__ void operator()(int64_t i, int64_t r, bool f) const {
    if (!f) return;
    uint64_t key = p.k[i];
    for (int q = 0; q < fs.d; ++q) {
      const uint64_t st = (uint64_t)fs.stride[q];
      coords[r * fs.d + q] = (int64_t)(key / st);
      key %= st;
    }
    vals[r] = p.run_sum(i);
  }
};

int bit_length(uint64_t x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

// Shared driver for the per-pass onesweep kernels once keys + histograms
// exist.  keys[0]/vals[0] hold the input; the result pointer is returned in
// *kres / *vres (one of the two ping-pong buffers).
// kin/vin (optional): the first executed pass reads these instead of
// keys[0]/vals[0]; kout/vout (optional): the last executed pass writes there
// (no staging copies in or out of the ping-pong buffers).
template <class MkDigit>
int onesweep_passes_t(ftt_ctx *ctx, uint64_t *keys[2], uint32_t *vals[2], int64_t n, int num_passes,
                      uint32_t *ghist, uint32_t *status, uint32_t *counters, uint64_t **kres,
                      uint32_t **vres, const uint64_t *kin, const uint32_t *vin, uint64_t *kout,
                      uint32_t *vout, MkDigit mk, bool all_active = false) {
  // decide which passes are needed (constant digit -> skip); hashed digits
  // (all_active) are never constant on inputs that reach this path, so their
  // histogram is not brought to the host (one round trip less)
  static thread_local std::vector<uint32_t> h;
  h.assign((size_t)num_passes * RADIX, 0);
  if (!all_active)
    FTT_CHECK(copy_to_host(ctx, h.data(), ghist, sizeof(uint32_t) * num_passes * RADIX));
  k_hist_scan<<<num_passes, RADIX, 0, ctx->stream>>>(ghist);
  FTT_LAUNCHED(ctx);
  // tile: RS_ITEMS = 16 keys per thread (measured on config 5: 8 / 12 / 24
  // items per thread were 13 % / 50 % / 140 % slower per pass)
  const int tile = RS_TILE;
  int64_t ntiles = ceil_div(n, tile);
  std::vector<int> active;
  for (int p = 0; p < num_passes; ++p) {
    bool trivial = false;
    for (int b = 0; b < RADIX; ++b)
      if ((int64_t)h[(size_t)p * RADIX + b] == n) trivial = true;
    if (!trivial) active.push_back(p);
  }
  const bool has_vals = vals[0] != nullptr;
  if (active.empty()) {  // already ordered: the input is the result
    if (kin && kout) {
      FTT_CUDA(cudaMemcpyAsync(kout, kin, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
      if (has_vals && vin && vout)
        FTT_CUDA(cudaMemcpyAsync(vout, vin, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
      *kres = kout;
      *vres = has_vals ? (vout ? vout : const_cast<uint32_t *>(vin)) : nullptr;
    } else {
      *kres = kin ? const_cast<uint64_t *>(kin) : keys[0];
      *vres = has_vals ? (vin ? const_cast<uint32_t *>(vin) : vals[0]) : nullptr;
    }
    return FTT_OK;
  }
  // one look-back status region per executed pass (<= 8), cleared at once
  FTT_CUDA(cudaMemsetAsync(status, 0, sizeof(uint32_t) * active.size() * ntiles * RADIX, ctx->stream));
  FTT_CUDA(cudaMemsetAsync(counters, 0, sizeof(uint32_t) * 8, ctx->stream));
  int cur = 0;
  const uint64_t *ksrc = kin ? kin : keys[0];
  const uint32_t *vsrc = vin ? vin : vals[0];
  for (size_t a = 0; a < active.size(); ++a) {
    const int p = active[a];
    const bool last = a + 1 == active.size();
    uint64_t *kdst = (last && kout) ? kout : keys[cur ^ 1];
    uint32_t *vdst = has_vals ? ((last && vout) ? vout : vals[cur ^ 1]) : nullptr;
    uint32_t *st = status + a * ntiles * RADIX;
    using DG = decltype(mk(0));
    static bool attr_set = false;
    // TMA prefetch: keys-only passes (3 CTAs / SM fit); passes with a
    // payload need 96 KB and run 2 CTAs / SM, measured slower than the
    // 3-CTA non-persistent pass (FTT_TMA_SORT=all forces them)
    static const char *tma_env = getenv("FTT_TMA_SORT");
    static const bool tma_off = tma_env && !strcmp(tma_env, "off");
    static const bool tma_all = tma_env && !strcmp(tma_env, "all");
    const bool use_tma = !tma_off && (!has_vals || tma_all);
    if (!attr_set) {
      const cudaFuncAttribute at = cudaFuncAttributeMaxDynamicSharedMemorySize;
      FTT_CUDA(cudaFuncSetAttribute(k_onesweep<true, RS_ITEMS, DG>, at, 12 * RS_TILE));
      FTT_CUDA(cudaFuncSetAttribute(k_onesweep<false, RS_ITEMS, DG>, at, 12 * RS_TILE));
      FTT_CUDA(cudaFuncSetAttribute(k_onesweep_tma<true, DG>, at, 24 * RS_TILE));
      FTT_CUDA(cudaFuncSetAttribute(k_onesweep_tma<false, DG>, at, 16 * RS_TILE));
      attr_set = true;
    }
    const int pb = prof_begin(ctx);
    // persistent: two CTAs per SM, each prefetching its next tile by TMA
    const bool aligned = ((uintptr_t)ksrc % 16 == 0) && (!has_vals || (uintptr_t)vsrc % 16 == 0);
    if (use_tma && aligned && ntiles > 2 * (int64_t)ctx->num_sms) {
      const unsigned grid =
          (unsigned)std::min<int64_t>(ntiles, (has_vals ? 2 : 3) * (int64_t)ctx->num_sms);
      if (has_vals)
        k_onesweep_tma<true, DG><<<grid, RS_THREADS, 24 * RS_TILE, ctx->stream>>>(
            ksrc, vsrc, kdst, vdst, n, mk(p), ghist + p * RADIX, st, counters + p, ntiles);
      else
        k_onesweep_tma<false, DG><<<grid, RS_THREADS, 16 * RS_TILE, ctx->stream>>>(
            ksrc, nullptr, kdst, nullptr, n, mk(p), ghist + p * RADIX, st, counters + p, ntiles);
    } else if (has_vals) {
      k_onesweep<true, RS_ITEMS, DG><<<(unsigned)ntiles, RS_THREADS, 12 * RS_TILE, ctx->stream>>>(
          ksrc, vsrc, kdst, vdst, n, mk(p), ghist + p * RADIX, st, counters + p);
    } else {
      k_onesweep<false, RS_ITEMS, DG><<<(unsigned)ntiles, RS_THREADS, 8 * RS_TILE, ctx->stream>>>(
          ksrc, nullptr, kdst, nullptr, n, mk(p), ghist + p * RADIX, st, counters + p);
    }
    FTT_LAUNCHED(ctx);
    // algorithmic bytes: read + write every key (and payload) once
    prof_end(ctx, pb, PT_SORT, (double)n * (has_vals ? 24.0 : 16.0), 0.0);
    ksrc = kdst;
    vsrc = vdst;
    cur ^= 1;
  }
  *kres = const_cast<uint64_t *>(ksrc);
  *vres = has_vals ? const_cast<uint32_t *>(vsrc) : nullptr;
  return FTT_OK;
}

int onesweep_passes(ftt_ctx *ctx, uint64_t *keys[2], uint32_t *vals[2], int64_t n, int num_passes,
                    uint32_t *ghist, uint32_t *status, uint32_t *counters, uint64_t **kres,
                    uint32_t **vres, const uint64_t *kin, const uint32_t *vin, uint64_t *kout,
                    uint32_t *vout) {
  return onesweep_passes_t(ctx, keys, vals, n, num_passes, ghist, status, counters, kres, vres, kin,
                           vin, kout, vout, [](int p) { return DigitShift{8 * p}; });
}

size_t onesweep_scratch(int64_t n) {
  int64_t ntiles = ceil_div(n, RS_MIN_TILE);
  return align_up(sizeof(uint32_t) * 8 * RADIX) + align_up(sizeof(uint32_t) * 8 * ntiles * RADIX) +
         align_up(sizeof(uint32_t) * 8);
}

int check_dims(int32_t d, const int64_t *dims, int32_t pivot, bool need_pivot) {
  if (d < 1 || d > 32) {
    set_error("number of modes %d out of range 1..32", d);
    return FTT_ERR_INVALID;
  }
  if (need_pivot && (pivot < 0 || pivot >= d)) {
    set_error("pivot %d out of range for %d modes", pivot, d);
    return FTT_ERR_INVALID;
  }
  __int128 size = 1;
  for (int k = 0; k < d; ++k) {
    if (dims[k] < 1) {
      set_error("shape extents must be positive");
      return FTT_ERR_INVALID;
    }
    size *= dims[k];
    if (size >= ((__int128)1 << 63)) {
      set_error("shape overflows 64-bit indexing");
      return FTT_ERR_INVALID;
    }
  }
  return FTT_OK;
}

// Key multipliers: mixed radix over the non-pivot modes in order, then the
// pivot as the fastest digit (include_pivot) or dropped.
void make_spec(int32_t d, const int64_t *dims, int32_t pivot, bool include_pivot, KeySpec *spec,
               uint64_t *key_bound) {
  spec->d = d;
  uint64_t m = include_pivot ? (uint64_t)dims[pivot] : 1;
  for (int k = d - 1; k >= 0; --k) {
    if (k == pivot) continue;
    spec->mult[k] = (int64_t)m;
    m *= (uint64_t)dims[k];
  }
  spec->mult[pivot] = include_pivot ? 1 : 0;
  *key_bound = m;  // keys < m
}

}  // namespace

size_t radix_sort_scratch_bytes(int64_t n, bool with_vals) {
  return onesweep_scratch(n) + 2 * align_up(sizeof(uint64_t) * n) +
         (with_vals ? 2 * align_up(sizeof(uint32_t) * n) : 0);
}

// Sort keys_in (+vals_in) over bits [0, end_bit); outputs into keys_out /
// vals_out (distinct from the inputs).  Arena must hold
// radix_sort_scratch_bytes(n).
int radix_sort(ftt_ctx *ctx, const uint64_t *keys_in, const uint32_t *vals_in, uint64_t *keys_out,
               uint32_t *vals_out, int64_t n, int end_bit) {
  if (n <= 0) return FTT_OK;
  int num_passes = (end_bit + 7) / 8;
  if (num_passes < 1) num_passes = 1;
  uint32_t *ghist = take<uint32_t>(ctx, 8 * RADIX);
  uint32_t *status = take<uint32_t>(ctx, 8 * ceil_div(n, RS_MIN_TILE) * RADIX);
  uint32_t *counters = take<uint32_t>(ctx, 8);
  uint64_t *kb[2] = {take<uint64_t>(ctx, n), take<uint64_t>(ctx, n)};
  uint32_t *vb[2] = {nullptr, nullptr};
  if (vals_in) {
    vb[0] = take<uint32_t>(ctx, n);
    vb[1] = take<uint32_t>(ctx, n);
  }
  if (!ghist || !status || !counters || !kb[0] || !kb[1] || (vals_in && (!vb[0] || !vb[1]))) {
    set_error("radix_sort: arena reservation too small");
    return FTT_ERR_INVALID;
  }
  FTT_CUDA(cudaMemsetAsync(ghist, 0, sizeof(uint32_t) * 8 * RADIX, ctx->stream));
  k_hist<<<grid_for(n, 256, 8), 256, 0, ctx->stream>>>(keys_in, n, num_passes, ghist, nullptr);
  FTT_LAUNCHED(ctx);
  // first pass reads the caller's arrays, last pass writes the caller's
  uint64_t *kr;
  uint32_t *vr;
  // (an in-place call keeps the staging: a pass must not scatter into the
  // array it reads)
  uint64_t *ko = keys_out == keys_in ? nullptr : keys_out;
  uint32_t *vo = (vals_out && vals_out == vals_in) ? nullptr : vals_out;
  FTT_CHECK(onesweep_passes(ctx, kb, vb, n, num_passes, ghist, status, counters, &kr, &vr, keys_in,
                            vals_in, ko, vo));
  if (kr != keys_out)
    FTT_CUDA(cudaMemcpyAsync(keys_out, kr, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  if (vals_out && vr && vr != vals_out)
    FTT_CUDA(cudaMemcpyAsync(vals_out, vr, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  return FTT_OK;
}

int sum_squares(ftt_ctx *ctx, int64_t n, const double *x, double *partial, double *out_host) {
  FTT_CHECK(sum_squares_dev(ctx, n, x, partial, partial + kSumSqBlocks));
  return copy_to_host(ctx, out_host, partial + kSumSqBlocks, sizeof(double));
}

// The same, leaving the total in device memory (*out_dev; 0 for n <= 0).
int dot_dev(ftt_ctx *ctx, int64_t n, const double *x, const double *y, double *partial,
            double *out_dev) {
  if (n <= 0) {
    FTT_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double), ctx->stream));
    return FTT_OK;
  }
  int nb = grid_for(n, 256, 4, kSumSqBlocks);
  k_dot_partial<<<nb, 256, 0, ctx->stream>>>(n, x, y, partial, out_dev, ctx->tile_cnt + kTileCnt);
  FTT_LAUNCHED(ctx);
  return FTT_OK;
}

int sum_squares_dev(ftt_ctx *ctx, int64_t n, const double *x, double *partial, double *out_dev) {
  if (n <= 0) {
    FTT_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double), ctx->stream));
    return FTT_OK;
  }
  int nb = grid_for(n, 256, 4, kSumSqBlocks);
  k_dot_partial<<<nb, 256, 0, ctx->stream>>>(n, x, nullptr, partial, out_dev,
                                             ctx->tile_cnt + kTileCnt);
  FTT_LAUNCHED(ctx);
  return FTT_OK;
}

int scan_block_counts(ftt_ctx *ctx, int64_t *counts, int64_t nblocks, int64_t *total_dev) {
  k_scan_counts<<<1, 1024, 0, ctx->stream>>>(counts, nblocks, total_dev);
  FTT_LAUNCHED(ctx);
  return FTT_OK;
}

// Internal: build keys from coords for one pivot and sort them.  With
// include_pivot the key is the fiber key and a permutation payload rides
// along; without, only the fixed-tuple keys are sorted (fiber count).
static int sort_coords(ftt_ctx *ctx, const int64_t *coords, int64_t nnz, int32_t d,
                       const int64_t *dims, int32_t pivot, bool include_pivot, uint64_t **kres,
                       uint32_t **vres, uint64_t *key_bound) {
  KeySpec spec;
  make_spec(d, dims, pivot, include_pivot, &spec, key_bound);
  int end_bit = bit_length(*key_bound > 0 ? *key_bound - 1 : 0);
  int num_passes = (end_bit + 7) / 8;
  if (num_passes < 1) num_passes = 1;
  uint32_t *ghist = take<uint32_t>(ctx, 8 * RADIX);
  uint32_t *status = take<uint32_t>(ctx, 8 * ceil_div(nnz, RS_MIN_TILE) * RADIX);
  uint32_t *counters = take<uint32_t>(ctx, 8);
  uint64_t *kb[2] = {take<uint64_t>(ctx, nnz), take<uint64_t>(ctx, nnz)};
  uint32_t *vb[2] = {nullptr, nullptr};
  if (include_pivot) {
    vb[0] = take<uint32_t>(ctx, nnz);
    vb[1] = take<uint32_t>(ctx, nnz);
  }
  if (!ghist || !status || !counters || !kb[1] || (include_pivot && !vb[1])) {
    set_error("sort_coords: arena reservation too small");
    return FTT_ERR_INVALID;
  }
  FTT_CUDA(cudaMemsetAsync(ghist, 0, sizeof(uint32_t) * 8 * RADIX, ctx->stream));
  const int pb = prof_begin(ctx);
  k_keys_hist<<<grid_for(nnz, 256, 8), 256, 0, ctx->stream>>>(coords, nnz, spec, num_passes, kb[0],
                                                              vb[0], ghist);
  FTT_LAUNCHED(ctx);
  // read the COO coordinates, write one key (+ identity payload) per nonzero
  prof_end(ctx, pb, PT_HIST, (double)nnz * (8.0 * d + 8.0 + (include_pivot ? 4.0 : 0.0)), 0.0);
  return onesweep_passes(ctx, kb, vb, nnz, num_passes, ghist, status, counters, kres, vres, nullptr,
                         nullptr, nullptr, nullptr);
}

static size_t sort_coords_bytes(int64_t nnz, bool with_perm) {
  return onesweep_scratch(nnz) + 2 * align_up(8 * nnz) + (with_perm ? 2 * align_up(4 * nnz) : 0);
}

}  // namespace ftt

using namespace ftt;

namespace {

void magic_u63(uint64_t D, uint64_t *m, int *sh) {
  // floor(x / D) = mulhi(x, m) >> sh for all x < 2^63 (Granlund-Montgomery,
  // N = 63: m = floor(2^(63+l) / D) + 1 < 2^64, l = ceil(log2 D)); D = 1 -> sh = -1
  if (D <= 1) {
    *m = 0;
    *sh = -1;
    return;
  }
  int l = 0;
  while (((unsigned __int128)1 << l) < D) ++l;
  const unsigned __int128 num = (unsigned __int128)1 << (63 + l);
  *m = (uint64_t)(num / D + 1);
  *sh = l - 1;
}

// Grouped counts from sorted orders (k_group_count): pivots p >= d/2 use the
// canonical C order (groups = the p leading modes), p < d/2 the reversed
// order (groups = the d-1-p trailing modes; one radix sort), each retried in
// the other order on overflow.  done[p] marks the pivots counted.
int fiber_counts_grouped(ftt_ctx *ctx, const int64_t *coords, int64_t nnz, int32_t d,
                         const int64_t *dims, int64_t *counts_host, bool *done) {
  for (int p = 0; p < d; ++p) done[p] = false;
  static const bool off = getenv("FTT_NO_GROUPED") != nullptr;
  if (off || d < 2) return FTT_OK;
  int64_t wc[32], wr[32];
  {
    int64_t st = 1;
    for (int k = d - 1; k >= 0; --k) {
      wc[k] = st;
      st *= dims[k];
    }
    st = 1;
    for (int k = 0; k < d; ++k) {
      wr[k] = st;
      st *= dims[k];
    }
  }
  uint64_t *lin = nullptr, *rlin = nullptr, *rsorted = nullptr;
  unsigned long long *cnt = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&lin, 8 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&cnt, 8 * 64 + 4 * 64 + 8));
  int *flags = reinterpret_cast<int *>(cnt + 64);
  int *unsorted = flags + 64;
  FTT_CUDA(cudaMemsetAsync(cnt, 0, 8 * 64 + 4 * 64 + 8, ctx->stream));
  LinSpec ls, rs;
  ls.d = rs.d = d;
  for (int k = 0; k < d; ++k) {
    ls.stride[k] = wc[k];
    rs.stride[k] = wr[k];
  }
  const bool need_rev = true;  // p = 0 always prefers the reversed order (d >= 2)
  FTT_CHECK(owned_alloc(ctx, (void **)&rlin, 8 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&rsorted, 8 * (size_t)nnz));
  int pb = prof_begin(ctx);
  k_linearize2<<<grid_for(nnz, 256, 4), 256, 0, ctx->stream>>>(coords, nnz, ls, rs, lin, rlin);
  FTT_LAUNCHED(ctx);
  // read the COO once, write both linear keys
  prof_end(ctx, pb, PT_HIST, (double)nnz * (8.0 * d + 16.0), 0.0);
  k_sorted_check<<<grid_for(nnz, 256, 8), 256, 0, ctx->stream>>>(lin, nnz, unsorted);
  FTT_LAUNCHED(ctx);
  {
    FTT_CHECK(arena_reserve(ctx, radix_sort_scratch_bytes(nnz, false) + 4096));
    uint64_t prod = 1;
    for (int k = 0; k < d; ++k) prod *= (uint64_t)dims[k];
    FTT_CHECK(radix_sort(ctx, rlin, nullptr, rsorted, nullptr, nnz, bit_length(prod - 1)));
    owned_free(ctx, rlin);
  }
  const unsigned nb = (unsigned)ceil_div(nnz, GC_L);
  static bool attr = false;
  if (!attr) {
    FTT_CUDA(cudaFuncSetAttribute(k_group_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  8 * GC_SLOTS));
    attr = true;
  }
  auto launch = [&](int p, bool rev, int slot) -> int {
    const uint64_t S = (uint64_t)(rev ? wr[p] : wc[p]);
    uint64_t mS, mT;
    int shS, shT;
    magic_u63(S, &mS, &shS);
    magic_u63(S * (uint64_t)dims[p], &mT, &shT);
    const int pb2 = prof_begin(ctx);
    k_group_count<<<nb, 256, 8 * GC_SLOTS, ctx->stream>>>(rev ? rsorted : lin, nnz, S, mS, shS, mT, shT,
                                               cnt + slot, flags + slot);
    FTT_LAUNCHED(ctx);
    prof_end(ctx, pb2, PT_SEGMENT, 8.0 * (double)nnz, 0.0);
    return FTT_OK;
  };
  // pass 1: preferred order (slots 0..d-1); pass 2: the other order (d..2d-1)
  for (int p = 0; p < d; ++p) FTT_CHECK(launch(p, 2 * p < d, p));
  unsigned long long h[64];
  int hf[64], hu = 0;
  FTT_CHECK(copy_to_host(ctx, h, cnt, 8 * 64));
  FTT_CHECK(copy_to_host(ctx, hf, flags, 4 * 64));
  FTT_CHECK(copy_to_host(ctx, &hu, unsorted, sizeof(int)));
  bool retried[32] = {false};
  bool retry = false;
  for (int p = 0; p < d; ++p) {
    const bool rev = 2 * p < d;
    const bool valid = !hf[p] && (rev || !hu);  // the C order needs sorted input
    if (valid) {
      counts_host[p] = (int64_t)h[p];
      done[p] = true;
      continue;
    }
    // the other order: C needs sorted input, the reversed order its sort
    const bool other_ok = rev ? !hu : need_rev;
    if (other_ok) {
      FTT_CHECK(launch(p, !rev, d + p));
      retried[p] = retry = true;
    }
  }
  if (retry) {
    FTT_CHECK(copy_to_host(ctx, h, cnt, 8 * 64));
    FTT_CHECK(copy_to_host(ctx, hf, flags, 4 * 64));
    for (int p = 0; p < d; ++p)
      if (retried[p] && !hf[d + p]) {
        counts_host[p] = (int64_t)h[d + p];
        done[p] = true;
      }
  }
  owned_free(ctx, lin);
  if (rsorted) owned_free(ctx, rsorted);
  owned_free(ctx, cnt);
  return FTT_OK;
}

int fiber_counts_partition(ftt_ctx *ctx, const int64_t *coords, int64_t nnz, int32_t d,
                           const int64_t *dims, int64_t *counts_host, const bool *skip) {
  // One pivot per pass: the bucketed key array (~1.2 x 8 B x nnz) then stays
  // resident in L2 between the scatter and the count, so the scattered 8-byte
  // writes merge in L2 instead of reaching DRAM as partial sectors (measured
  // with 4 pivots per pass: 3.3x write and 6x read amplification).
  // Bucket bits: ~2048 keys per bucket on average; fixed capacity mean +
  // 8 sigma (+64): overflow (duplicate-heavy pivots) falls back to sorting
  int bits = 4;
  while (bits < 12 && (nnz >> bits) > 2048) ++bits;
  const int nbk = 1 << bits;
  const int64_t mean = ceil_div(nnz, nbk);
  // (fibers with several nonzeros land whole in one bucket: the variance of a
  // bucket's fill is ~mean x (average fiber size), hence the wide margin)
  const int64_t cap = std::min<int64_t>(nnz, mean + 16 * (int64_t)std::sqrt((double)mean) + 256);
  const int G = 1;  // pivots per pass (more per pass measured no faster)
  const int nb = kNumSMs;
  LinSpec ls;
  ls.d = d;
  {
    int64_t st = 1;
    for (int k = d - 1; k >= 0; --k) {
      ls.stride[k] = st;
      st *= dims[k];
    }
  }
  uint64_t *lin = nullptr, *keys = nullptr;
  unsigned int *fill = nullptr;
  unsigned long long *cnt = nullptr;
  int *flags = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&lin, 8 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&keys, 8 * (size_t)cap * nbk * G));
  FTT_CHECK(owned_alloc(ctx, (void **)&fill, 4 * (size_t)G * nbk * ceil_div(d, G)));
  FTT_CHECK(owned_alloc(ctx, (void **)&cnt, 8 * 32 + 4 * 32));
  flags = reinterpret_cast<int *>(cnt + 32);
  FTT_CUDA(cudaMemsetAsync(cnt, 0, 8 * 32 + 4 * 32, ctx->stream));
  FTT_CUDA(cudaMemsetAsync(fill, 0, 4 * (size_t)G * nbk * ceil_div(d, G), ctx->stream));
  static bool attrs = false;
  if (!attrs) {
    FTT_CUDA(cudaFuncSetAttribute(k_part_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  65536));
    FTT_CUDA(cudaFuncSetAttribute(k_part_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  8 * PC_TMAX));
    attrs = true;
  }
  int pb = prof_begin(ctx);
  k_linearize<<<grid_for(nnz, 256, 4), 256, 0, ctx->stream>>>(coords, nnz, ls, lin);
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb, PT_HIST, (double)nnz * (8.0 * d + 8.0), 0.0);
  for (int p0 = 0, grp = 0; p0 < d; p0 += G, ++grp) {
    if (G == 1 && skip && skip[p0]) continue;  // counted by the grouped path
    PartSpec ps;
    ps.g = std::min(G, d - p0);
    ps.bits = bits;
    ps.chunk = ceil_div(nnz, nb);
    for (int q = 0; q < ps.g; ++q) {
      const int p = p0 + q;
      const uint64_t S = (uint64_t)ls.stride[p];
      ps.S[q] = S;
      magic_u63(S, &ps.mS[q], &ps.shS[q]);
      magic_u63(S * (uint64_t)dims[p], &ps.mT[q], &ps.shT[q]);
    }
    const int tot = ps.g * nbk;
    unsigned int *gfill = fill + (size_t)grp * G * nbk;
    pb = prof_begin(ctx);
    k_part_scatter<<<nb, 1024, 4 * (size_t)tot, ctx->stream>>>(lin, nnz, ps, cap, gfill, keys,
                                                               flags + p0);
    FTT_LAUNCHED(ctx);
    // read lin (the second read of each chunk hits L2), write one key per pivot
    prof_end(ctx, pb, PT_SORT, (double)nnz * (8.0 + 8.0 * ps.g), 0.0);
    pb = prof_begin(ctx);
    k_part_count<<<dim3(nbk, ps.g), 256, 8 * PC_TMAX, ctx->stream>>>(keys, cap, gfill, nbk,
                                                                      cnt + p0, flags + p0);
    FTT_LAUNCHED(ctx);
    prof_end(ctx, pb, PT_SEGMENT, 8.0 * (double)nnz * ps.g, 0.0);
  }
  unsigned long long h[32];
  int hf[32];
  FTT_CHECK(copy_to_host(ctx, h, cnt, 8 * 32));
  FTT_CHECK(copy_to_host(ctx, hf, flags, 4 * 32));
  owned_free(ctx, lin);
  owned_free(ctx, keys);
  owned_free(ctx, fill);
  owned_free(ctx, cnt);
  static const bool debug = getenv("FTT_DEBUG") != nullptr;
  for (int p = 0; p < d; ++p) {
    if (G == 1 && skip && skip[p]) continue;
    if (debug && hf[p]) fprintf(stderr, "[ftt] select_p partition overflow at pivot %d\n", p);
    if (hf[p]) FTT_CHECK(ftt_fiber_count(ctx, coords, nnz, d, dims, p, &counts_host[p]));
    else counts_host[p] = (int64_t)h[p];
  }
  return FTT_OK;
}

}  // namespace

namespace ftt {
namespace {

// ---- select_p counts and fiber keys from the canonical linear index -----
// The device COO is kept as its C-order linear index `lin` (8 B per nonzero,
// strictly increasing: SparseTensor's canonical form) plus the values; every
// digit a kernel needs is an exact magic-number division of lin.
//
// select_p counts (fasttt.py:536-541) per pivot p = distinct fixed tuples
// (lin with digit p removed).  With pf = ceil(d / 2) and M = prod dims[pf:]:
//  * pivots p >= pf: nonzeros sharing a fixed tuple share the prefix over
//    modes < p, hence lin / M; chunks of lin aligned to lin / M groups hold
//    whole fibers of all those pivots at once (one read, no sort);
//  * pivots p < pf: they share lin mod M (the suffix over modes >= pf);
//    lin is bucketed by h = mix64(lin mod M) >> 48 (two stable radix passes
//    on digits of h, keys only) and chunks are aligned to h runs.
// In a chunk, each pivot's fixed-tuple keys go into a shared-memory hash set
// -- 32-bit keys relative to the chunk minimum when the chunk's key span fits
// (a single CAS per insert), else 64-bit -- and first insertions are
// counted: exact and independent of the insertion order.  A group longer
// than the chunk capacity flags its pivots (the caller counts those another
// way); unsorted input flags the lin-order pivots.
constexpr int SC_L = 1024;       // nominal nonzeros per CTA (groups up to SC_CAP - SC_L)
constexpr int SC_CAP = 4096;     // max nonzeros per chunk
constexpr int SC_SLOTS = 8192;   // 32-bit hash slots (load <= 1/2)
constexpr int SC_MAXP = 32;
constexpr int SC_NT = 512;      // threads per chunk CTA

struct SelSpec {
  int np;
  int align_hash;  // 0: group = lin / M; 1: group = mix64(lin mod M) >> 48
  uint64_t M, mM;
  int shM;
  int lgM;  // log2 M when every extent is a power of two (shift / mask keys)
  int lgS[SC_MAXP], lgT[SC_MAXP];
  uint64_t S[SC_MAXP], mS[SC_MAXP], mT[SC_MAXP];
  int shS[SC_MAXP], shT[SC_MAXP], slot[SC_MAXP];
};

template <bool POW2>
__device__ __forceinline__ uint64_t sel_group(uint64_t x, const SelSpec &sp) {
  if (POW2) {
    if (!sp.align_hash) return x >> sp.lgM;
    return mix64(x & ((1ull << sp.lgM) - 1)) >> 48;
  }
  const uint64_t q = udiv_magic(x, sp.mM, sp.shM);
  if (!sp.align_hash) return q;
  return mix64(x - q * sp.M) >> 48;
}

struct DigitHashMod {  // bits [shift, shift + 8) of mix64(lin mod M) >> 48
  uint64_t M, mM;
  int shM, shift;
  __device__ __forceinline__ uint32_t operator()(uint64_t k) const {
    const uint64_t lo = k - udiv_magic(k, mM, shM) * M;
    return (uint32_t)(((mix64(lo) >> 48) >> shift) & 255);
  }
};

__global__ void __launch_bounds__(256) k_hist_hashmod(const uint64_t *__restrict__ keys, int64_t n,
                                                      DigitHashMod dg, uint32_t *__restrict__ ghist) {
  __shared__ uint32_t sh[2][RADIX];
  for (int i = threadIdx.x; i < 2 * RADIX; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    const uint64_t lo = k - udiv_magic(k, dg.mM, dg.shM) * dg.M;
    const uint32_t h = (uint32_t)(mix64(lo) >> 48);
    atomicAdd(&sh[0][h & 255], 1u);
    atomicAdd(&sh[1][h >> 8], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * RADIX; i += blockDim.x) {
    const uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(&ghist[i], v);
  }
}

template <bool POW2>
__global__ void __launch_bounds__(SC_NT) k_sel_count(const uint64_t *__restrict__ K, int64_t n,
                                                   SelSpec sp,
                                                   unsigned long long *__restrict__ count,
                                                   int *__restrict__ flag,
                                                   int *__restrict__ unsorted, unsigned blk_off) {
  extern __shared__ unsigned long long smem[];
  // the chunk's keys stay in global memory: at most 32 KB per CTA, re-read
  // through L1 by every pivot's pass; shared memory holds only the table
  // (32 KB: 4 CTAs per SM)
  unsigned *tab32 = reinterpret_cast<unsigned *>(smem);   // SC_SLOTS positions
  __shared__ int64_t s_start, s_end;
  __shared__ unsigned s_j[2];
  __shared__ unsigned s_cnt;  // first insertions of one pivot in this chunk (<= SC_CAP)
  const int lane = threadIdx.x & 31;
  const int64_t c0 = ((int64_t)blockIdx.x + blk_off) * SC_L;
  auto grp = [&](int64_t i) -> uint64_t { return sel_group<POW2>(K[i], sp); };
  if (threadIdx.x < 2) s_j[threadIdx.x] = 0xffffffffu;
  __syncthreads();
  // chunk = whole groups starting in [c0, c0 + L): first group start at or
  // after c0 and at or after c0 + L (both windows searched together)
  bool open0 = c0 < n, open1 = c0 + SC_L < n;
  for (int r = 0; r < SC_CAP / SC_NT && (open0 || open1); ++r) {
    const int j = r * SC_NT + (int)threadIdx.x;
    bool st0 = false, st1 = false;
    if (open0) {
      const int64_t i = c0 + j;
      st0 = i <= n && (i == n || i == 0 || grp(i) != grp(i - 1));
    }
    if (open1) {
      const int64_t i = c0 + SC_L + j;
      st1 = i <= n && (i == n || grp(i) != grp(i - 1));
    }
    const unsigned m0 = __reduce_min_sync(0xffffffffu, st0 ? (unsigned)j : 0xffffffffu);
    const unsigned m1 = __reduce_min_sync(0xffffffffu, st1 ? (unsigned)j : 0xffffffffu);
    if (lane == 0 && m0 != 0xffffffffu) atomicMin(&s_j[0], m0);
    if (lane == 0 && m1 != 0xffffffffu) atomicMin(&s_j[1], m1);
    const int any0 = __syncthreads_or(st0);
    const int any1 = __syncthreads_or(st1);
    open0 = open0 && !any0;
    open1 = open1 && !any1;
  }
  if (threadIdx.x == 0) {
    s_start = c0 >= n ? n : (s_j[0] == 0xffffffffu ? INT64_MAX : c0 + s_j[0]);
    s_end = c0 + SC_L >= n ? n : (s_j[1] == 0xffffffffu ? INT64_MAX : c0 + SC_L + s_j[1]);
  }
  __syncthreads();
  const int64_t start = s_start, end = s_end;
  if (start == INT64_MAX) return;  // inside a long group: its owner flags it
  if (end == INT64_MAX || end - start > SC_CAP) {
    if (threadIdx.x == 0)
      for (int q = 0; q < sp.np; ++q) atomicOr(flag + sp.slot[q], 1);
    return;
  }
  constexpr int PER = SC_CAP / SC_NT;
  const int cnt = (int)(end - start);
  int bad = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = q * SC_NT + threadIdx.x;
    if (j < cnt) {
      if (!sp.align_hash && start + j + 1 < n) bad |= __ldg(K + start + j + 1) <= __ldg(K + start + j);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(unsorted, 1);
  const uint64_t *__restrict__ skey = K + start;
  // per pivot: the table holds chunk positions (native 32-bit shared CAS);
  // a probe that meets an occupied slot compares the fixed-tuple key of the
  // stored position, recomputed from its lin
  for (int q = 0; q < sp.np; ++q) {
    const uint64_t S = sp.S[q];
    const uint64_t mT = sp.mT[q], mS = sp.mS[q];
    const int shT = sp.shT[q], shS = sp.shS[q], lgS = sp.lgS[q], lgT = sp.lgT[q];
    auto reduce = [&](uint64_t x) -> uint64_t {
      if (POW2) return ((x >> lgT) << lgS) | (x & ((1ull << lgS) - 1));
      return udiv_magic(x, mT, shT) * S + (x - udiv_magic(x, mS, shS) * S);
    };
    // multiplicative hash (Fibonacci), 13 bits
    auto slot = [](uint64_t k) -> unsigned {
      return (unsigned)((k * 0x9E3779B97F4A7C15ull) >> (64 - 13));
    };
    unsigned fresh = 0;
    if (!sp.align_hash && S == 1) {
      // last mode in lin order: a fiber's nonzeros are adjacent (the chunk is
      // sorted, else `unsorted` sends the caller to another count), so first
      // occurrences are adjacent differences -- no table
      for (int j = threadIdx.x; j < cnt; j += SC_NT)
        fresh += j == 0 || reduce(__ldg(skey + j - 1)) != reduce(__ldg(skey + j));
      fresh = __reduce_add_sync(0xffffffffu, fresh);
      if (lane == 0 && fresh) atomicAdd(count + sp.slot[q], (unsigned long long)fresh);
      continue;
    }
    for (int e = threadIdx.x; e < SC_SLOTS / 4; e += SC_NT)
      reinterpret_cast<uint4 *>(tab32)[e] = make_uint4(~0u, ~0u, ~0u, ~0u);
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += SC_NT) {  // only the chunk's live rounds
      const uint64_t r = reduce(__ldg(skey + j));
      unsigned h = slot(r);
      while (true) {
        const unsigned old = atomicCAS(tab32 + h, ~0u, (unsigned)j);
        if (old == ~0u) {
          ++fresh;
          break;
        }
        if (reduce(__ldg(skey + old)) == r) break;
        h = (h + 1) & (SC_SLOTS - 1);  // linear probing
      }
    }
    fresh = __reduce_add_sync(0xffffffffu, fresh);
    if (lane == 0 && fresh) atomicAdd(&s_cnt, fresh);
    __syncthreads();
    if (threadIdx.x == 0 && s_cnt) atomicAdd(count + sp.slot[q], (unsigned long long)s_cnt);
  }
}

// Fiber keys straight from lin: key = fixed_lin = (lin / T) * S + lin mod S
// (S = prod of the dims after the pivot, T = n_p S), identity payload, digit
// histograms of every pass.  The pivot index is NOT in the key: lin order is
// (prefix, i_p, suffix), so a STABLE sort by the fixed tuple alone leaves
// equal tuples in ascending i_p -- the reference's lexsort order
// (tensor.py:387-389) with log2(n_p) fewer key bits (config 5: 55 bits, 7
// passes instead of 8).  Reads 8 B per nonzero instead of the d coordinates.
struct LinKeySpec {
  uint64_t S, mS, T, mT, np, mN;
  int shS, shT, shN;
};

__device__ __forceinline__ uint64_t lin_fiber_key(uint64_t x, const LinKeySpec &ks, uint64_t *ip) {
  const uint64_t a = udiv_magic(x, ks.mS, ks.shS);  // lin / S
  const uint64_t lo = x - a * ks.S;
  const uint64_t hi = udiv_magic(x, ks.mT, ks.shT);  // lin / T
  if (ip) *ip = a - hi * ks.np;
  return hi * ks.S + lo;
}

// Emit of the fiber extraction on the fixed-tuple keys: the pivot index is
// re-derived from lin[perm[i]] (a gather from the chunk the sort just read).
// Two-phase form (kTwoPhase): k_compact1 first loads the gathers of a batch
// of items (perm -> lin, value: two dependent random reads per nonzero) and
// only then stores -- interleaved with the stores, as operator() has them,
// the loads of the next item cannot be hoisted (the outputs may alias) and
// the kernel ran one gather chain per thread at a time (ncu: 16 % issue
// active, long-scoreboard stalls).
struct FiberEmitLin {
  static constexpr bool kTwoPhase = true;
  struct Item {
    uint64_t key, lin;
    double val;
  };
  __device__ Item load(int64_t i) const {
    const uint32_t src = __ldg(perm + i);
    Item it;
    it.key = __ldg(k + i);
    it.lin = __ldg(lin + src);
    it.val = __ldg(vals_in + src);
    return it;
  }
  __device__ void store(int64_t i, int64_t r, bool f, const Item &it) const {
    if (f) {
      indptr[r] = i;
      fixed_lin[r] = (int64_t)it.key;
    }
    if (fiber_of) fiber_of[i] = f ? r : r - 1;
    uint64_t ip = 0;
    lin_fiber_key(it.lin, ks, &ip);
    pivot_index[i] = (int64_t)ip;
    vals_out[i] = it.val;
  }
  const uint64_t *k;
  const uint32_t *perm;
  const double *vals_in;
  const uint64_t *lin;
  LinKeySpec ks;
  int64_t *fixed_lin, *indptr, *fiber_of, *pivot_index;
  double *vals_out;
};

__global__ void __launch_bounds__(256) k_keys_hist_lin(const uint64_t *__restrict__ lin, int64_t n,
                                                       LinKeySpec ks, int num_passes,
                                                       uint64_t *__restrict__ keys,
                                                       uint32_t *__restrict__ idx,
                                                       uint32_t *__restrict__ ghist) {
  __shared__ uint32_t sh[8][RADIX];
  for (int i = threadIdx.x; i < 8 * RADIX; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = lin_fiber_key(lin[i], ks, nullptr);
    keys[i] = key;
    idx[i] = (uint32_t)i;
    for (int p = 0; p < num_passes; ++p) atomicAdd(&sh[p][(key >> (8 * p)) & 255], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < num_passes * RADIX; i += blockDim.x) {
    const uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(&ghist[i], v);
  }
}

__global__ void k_linearize_c(const int64_t *__restrict__ coords, int64_t n, LinSpec ls,
                              int64_t *__restrict__ lin) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t *c = coords + i * ls.d;
    uint64_t x = 0;
    for (int k = 0; k < ls.d; ++k) x += (uint64_t)c[k] * (uint64_t)ls.stride[k];
    lin[i] = (int64_t)x;
  }
}

void c_strides(int32_t d, const int64_t *dims, int64_t *w) {
  int64_t st = 1;
  for (int k = d - 1; k >= 0; --k) {
    w[k] = st;
    st *= dims[k];
  }
}

// Counts for every pivot from lin; done[p] false where the caller must
// count pivot p another way (a group over capacity, or unsorted input).
int fiber_counts_lin(ftt_ctx *ctx, const uint64_t *lin, int64_t nnz, int32_t d, const int64_t *dims,
                     int64_t *counts_host, bool *done) {
  for (int p = 0; p < d; ++p) done[p] = false;
  if (d < 2) return FTT_OK;
  int64_t w[32];
  c_strides(d, dims, w);
  const int pf = (d + 1) / 2;
  const uint64_t M = (uint64_t)w[pf - 1];  // prod dims[pf:]
  SelSpec fwd, rev;
  fwd.align_hash = 0;
  rev.align_hash = 1;
  fwd.M = rev.M = M;
  magic_u63(M, &fwd.mM, &fwd.shM);
  rev.mM = fwd.mM;
  rev.shM = fwd.shM;
  fwd.np = rev.np = 0;
  bool pow2 = true;
  for (int p = 0; p < d; ++p) pow2 &= (dims[p] & (dims[p] - 1)) == 0;
  auto lg2 = [](uint64_t x) {
    int l = 0;
    while ((1ull << l) < x) ++l;
    return l;
  };
  fwd.lgM = rev.lgM = pow2 ? lg2(M) : 0;
  for (int p = 0; p < d; ++p) {
    SelSpec &sp = p >= pf ? fwd : rev;
    const int q = sp.np++;
    sp.S[q] = (uint64_t)w[p];
    magic_u63((uint64_t)w[p], &sp.mS[q], &sp.shS[q]);
    magic_u63((uint64_t)w[p] * (uint64_t)dims[p], &sp.mT[q], &sp.shT[q]);
    sp.lgS[q] = pow2 ? lg2((uint64_t)w[p]) : 0;
    sp.lgT[q] = pow2 ? lg2((uint64_t)w[p] * (uint64_t)dims[p]) : 0;
    sp.slot[q] = p;
  }
  unsigned long long *cnt = nullptr;
  uint64_t *bucketed = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&cnt, 8 * 32 + 4 * 32 + 16));
  int *flags = reinterpret_cast<int *>(cnt + 32);
  int *unsorted = flags + 32;
  FTT_CUDA(cudaMemsetAsync(cnt, 0, 8 * 32 + 4 * 32 + 16, ctx->stream));
  static bool attr = false;
  const size_t smem = 4 * (size_t)SC_SLOTS;
  if (!attr) {
    FTT_CUDA(cudaFuncSetAttribute(k_sel_count<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    FTT_CUDA(cudaFuncSetAttribute(k_sel_count<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr = true;
  }
  const unsigned nb = (unsigned)ceil_div(nnz, SC_L);
  auto count = [&](const uint64_t *keys, const SelSpec &sp, int *uns, unsigned b0, unsigned b1) {
    if (b1 <= b0) return;
    if (pow2)
      k_sel_count<true><<<b1 - b0, SC_NT, smem, ctx->stream>>>(keys, nnz, sp, cnt, flags, uns, b0);
    else
      k_sel_count<false><<<b1 - b0, SC_NT, smem, ctx->stream>>>(keys, nnz, sp, cnt, flags, uns, b0);
  };
  int pb = prof_begin(ctx);
  {
    // lin may still be arriving from the host in chunks (ftt_set_lin_chunks):
    // the forward counts of the blocks whose window (SC_L + the SC_CAP
    // look-ahead + 1) lies inside the chunks present start at once
    const int nch = ctx->lin_nchunks;
    ctx->lin_nchunks = 0;
    unsigned b0 = 0;
    for (int j = 0; j < nch; ++j) {
      FTT_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->lin_events[j], 0));
      const int64_t have = std::min<int64_t>(ctx->lin_ends[j], nnz);
      unsigned b1 = nb;
      if (j + 1 < nch && have < nnz) {
        const int64_t full = (have - SC_CAP - 1) / SC_L - 1;  // last block wholly covered
        b1 = (unsigned)std::max<int64_t>(b0, std::min<int64_t>(nb, full + 1));
      }
      count(lin, fwd, unsorted, b0, b1);
      b0 = b1;
    }
    count(lin, fwd, unsorted, b0, nb);
  }
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb, PT_SEGMENT, 8.0 * (double)nnz, 0.0);
  if (rev.np > 0) {
    // bucket lin by h = mix64(lin mod M) >> 48: two stable passes, keys only
    FTT_CHECK(owned_alloc(ctx, (void **)&bucketed, 8 * (size_t)nnz));
    FTT_CHECK(arena_reserve(ctx, onesweep_scratch(nnz) + 2 * align_up(8 * (size_t)nnz) + 4096));
    uint32_t *ghist = take<uint32_t>(ctx, 8 * RADIX);
    uint32_t *status = take<uint32_t>(ctx, 8 * ceil_div(nnz, RS_MIN_TILE) * RADIX);
    uint32_t *counters = take<uint32_t>(ctx, 8);
    uint64_t *kb[2] = {take<uint64_t>(ctx, nnz), take<uint64_t>(ctx, nnz)};
    uint32_t *vb[2] = {nullptr, nullptr};
    FTT_CUDA(cudaMemsetAsync(ghist, 0, sizeof(uint32_t) * 8 * RADIX, ctx->stream));
    DigitHashMod dg{M, fwd.mM, fwd.shM, 0};
    pb = prof_begin(ctx);
    k_hist_hashmod<<<grid_for(nnz, 256, 8), 256, 0, ctx->stream>>>(lin, nnz, dg, ghist);
    FTT_LAUNCHED(ctx);
    prof_end(ctx, pb, PT_HIST, 8.0 * (double)nnz, 0.0);
    uint64_t *kr = nullptr;
    uint32_t *vr = nullptr;
    FTT_CHECK(onesweep_passes_t(ctx, kb, vb, nnz, 2, ghist, status, counters, &kr, &vr, lin, nullptr,
                                bucketed, nullptr, [&](int p) {
                                  DigitHashMod g = dg;
                                  g.shift = 8 * p;
                                  return g;
                                },
                                /*all_active=*/true));
    pb = prof_begin(ctx);
    count(kr, rev, unsorted + 1, 0, nb);
    FTT_LAUNCHED(ctx);
    prof_end(ctx, pb, PT_SEGMENT, 8.0 * (double)nnz, 0.0);
  }
  unsigned long long h[32 + 17];  // counts, then the 34 flag words: one round trip
  FTT_CHECK(copy_to_host(ctx, h, cnt, 8 * 32 + 4 * 34));
  int hf[34];
  memcpy(hf, h + 32, 4 * 34);
  if (bucketed) owned_free(ctx, bucketed);
  owned_free(ctx, cnt);
  const bool sorted = hf[32] == 0;
  for (int p = 0; p < d; ++p) {
    if (hf[p] || (p >= pf && !sorted)) continue;
    counts_host[p] = (int64_t)h[p];
    done[p] = true;
  }
  return FTT_OK;
}

int fiber_keys_lin(ftt_ctx *ctx, const uint64_t *lin, int64_t nnz, int32_t d, const int64_t *dims,
                   int32_t pivot, uint64_t **kres, uint32_t **vres, LinKeySpec *spec_out) {
  int64_t w[32];
  c_strides(d, dims, w);
  LinKeySpec ks;
  ks.S = (uint64_t)w[pivot];
  ks.np = (uint64_t)dims[pivot];
  ks.T = ks.S * ks.np;
  magic_u63(ks.S, &ks.mS, &ks.shS);
  magic_u63(ks.T, &ks.mT, &ks.shT);
  magic_u63(ks.np, &ks.mN, &ks.shN);
  uint64_t bound = 1;  // fixed tuples < prod of the other extents
  for (int k = 0; k < d; ++k)
    if (k != pivot) bound *= (uint64_t)dims[k];
  *spec_out = ks;
  int num_passes = (bit_length(bound - 1) + 7) / 8;
  if (num_passes < 1) num_passes = 1;
  uint32_t *ghist = take<uint32_t>(ctx, 8 * RADIX);
  uint32_t *status = take<uint32_t>(ctx, 8 * ceil_div(nnz, RS_MIN_TILE) * RADIX);
  uint32_t *counters = take<uint32_t>(ctx, 8);
  uint64_t *kb[2] = {take<uint64_t>(ctx, nnz), take<uint64_t>(ctx, nnz)};
  uint32_t *vb[2] = {take<uint32_t>(ctx, nnz), take<uint32_t>(ctx, nnz)};
  if (!ghist || !status || !counters || !kb[1] || !vb[1]) {
    set_error("fiber_keys_lin: arena reservation too small");
    return FTT_ERR_INVALID;
  }
  FTT_CUDA(cudaMemsetAsync(ghist, 0, sizeof(uint32_t) * 8 * RADIX, ctx->stream));
  const int pb = prof_begin(ctx);
  k_keys_hist_lin<<<grid_for(nnz, 256, 8), 256, 0, ctx->stream>>>(lin, nnz, ks, num_passes, kb[0],
                                                                  vb[0], ghist);
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb, PT_HIST, (double)nnz * 20.0, 0.0);
  return onesweep_passes(ctx, kb, vb, nnz, num_passes, ghist, status, counters, kres, vres, nullptr,
                         nullptr, nullptr, nullptr);
}


}  // namespace
}  // namespace ftt

namespace {
}  // namespace

extern "C" {

int ftt_fiber_count(ftt_ctx *ctx, const int64_t *coords, int64_t nnz, int32_t d,
                    const int64_t *dims_host, int32_t pivot, int64_t *count_out) {
  if (!ctx || !count_out) return FTT_ERR_INVALID;
  FTT_CHECK(check_dims(d, dims_host, pivot, true));
  if (nnz >= ((int64_t)1 << 30)) {
    set_error("nnz %lld exceeds the 2^30 sort limit", (long long)nnz);
    return FTT_ERR_INVALID;
  }
  if (nnz == 0) {
    *count_out = 0;
    return FTT_OK;
  }
  FTT_CHECK(arena_reserve(ctx, sort_coords_bytes(nnz, false) + 1024));
  uint64_t *kr;
  uint32_t *vr;
  uint64_t bound;
  FTT_CHECK(sort_coords(ctx, coords, nnz, d, dims_host, pivot, false, &kr, &vr, &bound));
  unsigned long long *cnt = take<unsigned long long>(ctx, 1);
  FTT_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), ctx->stream));
  k_count_changes<<<grid_for(nnz, 256, 8), 256, 0, ctx->stream>>>(kr, nnz, cnt);
  FTT_LAUNCHED(ctx);
  unsigned long long h = 0;
  FTT_CHECK(copy_to_host(ctx, &h, cnt, sizeof(h)));
  *count_out = (int64_t)h;
  return FTT_OK;
}

int ftt_fiber_counts_all(ftt_ctx *ctx, const int64_t *coords, int64_t nnz, int32_t d,
                         const int64_t *dims_host, int64_t *counts_host) {
  if (!ctx || !counts_host) return FTT_ERR_INVALID;
  FTT_CHECK(check_dims(d, dims_host, 0, false));
  if (nnz >= ((int64_t)1 << 30)) {
    set_error("nnz exceeds the 2^30 sort limit");
    return FTT_ERR_INVALID;
  }
  if (nnz == 0) {
    for (int p = 0; p < d; ++p) counts_host[p] = 0;
    return FTT_OK;
  }
  // One pass over the COO: every nonzero inserts its d fixed-tuple keys into
  // d open-addressing hash sets (table size 2^ceil(log2(2 nnz))); a CAS that
  // claims an empty slot is a new distinct key.  Exact (insertion order does
  // not change the count) and reads the coordinates once instead of d
  // radix sorts.  Tables for all d pivots at once when they fit in 4 GiB,
  // else pivot groups.  Once one table outgrows a slice of L2 the random CAS
  // traffic goes to HBM and d onesweep sorts (streaming, coalesced) win, so
  // large inputs take the sort route (measured crossover ~2-4M nonzeros).
  int lg = 1;
  while (((int64_t)1 << lg) < 2 * nnz) ++lg;
  const int64_t T = (int64_t)1 << lg;
  const char *path = getenv("FTT_COUNT_PATH");  // test override: hash | part | sort
  const bool force_part = path && !strcmp(path, "part");
  const bool force_sort = path && !strcmp(path, "sort");
  const bool force_hash = path && !strcmp(path, "hash");
  const bool force_group = path && !strcmp(path, "group");
  if (force_sort) {
    for (int p = 0; p < d; ++p)
      FTT_CHECK(ftt_fiber_count(ctx, coords, nnz, d, dims_host, p, &counts_host[p]));
    return FTT_OK;
  }
  if (force_part)
    return fiber_counts_partition(ctx, coords, nnz, d, dims_host, counts_host, nullptr);
  if (force_group || (!force_hash && 8 * T > ((int64_t)32 << 20))) {
    // large inputs: group-local counts from the sorted orders first, the
    // bucket partition for any pivot whose groups are too long
    bool done[32];
    FTT_CHECK(fiber_counts_grouped(ctx, coords, nnz, d, dims_host, counts_host, done));
    bool all = true;
    for (int p = 0; p < d; ++p) all &= done[p];
    static const bool debug = getenv("FTT_DEBUG") != nullptr;
    if (debug)
      for (int p = 0; p < d; ++p)
        if (!done[p]) fprintf(stderr, "[ftt] select_p grouped count: pivot %d -> partition\n", p);
    if (all) return FTT_OK;
    return fiber_counts_partition(ctx, coords, nnz, d, dims_host, counts_host, done);
  }
  int group = (int)std::max<int64_t>(1, std::min<int64_t>(d, ((int64_t)1 << 29) / T));  // 4 GiB
  group = std::min(group, HS_PASS);
  uint64_t *tables = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&tables, 8 * (size_t)T * group));
  FTT_CHECK(arena_reserve(ctx, 4096));
  unsigned long long *cnt = take<unsigned long long>(ctx, 32);
  FTT_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * 32, ctx->stream));
  for (int p0 = 0; p0 < d; p0 += group) {
    const int np = std::min(group, d - p0);
    HashSpec hs;
    hs.d = d;
    hs.np = np;
    hs.lg = lg;
    {
      int64_t st = 1;
      for (int k = d - 1; k >= 0; --k) {
        hs.stride[k] = st;
        st *= dims_host[k];
      }
    }
    for (int q = 0; q < np; ++q) {
      const uint64_t S = (uint64_t)hs.stride[p0 + q];
      hs.S[q] = S;
      magic_u63(S, &hs.mS[q], &hs.shS[q]);
      magic_u63(S * (uint64_t)dims_host[p0 + q], &hs.mT[q], &hs.shT[q]);
    }
    FTT_CUDA(cudaMemsetAsync(tables, 0xff, 8 * (size_t)T * np, ctx->stream));
    const int pb = prof_begin(ctx);
    k_distinct_hash<<<grid_for(nnz, 256, 1), 256, 0, ctx->stream>>>(
        coords, nullptr, nnz, hs, reinterpret_cast<unsigned long long *>(tables), cnt + p0);
    FTT_LAUNCHED(ctx);
    // coordinates read once + one 8-byte CAS per pivot and nonzero
    prof_end(ctx, pb, PT_HIST, (double)nnz * (8.0 * d + 8.0 * np), 0.0);
  }
  owned_free(ctx, tables);
  unsigned long long h[32];
  FTT_CHECK(copy_to_host(ctx, h, cnt, sizeof(unsigned long long) * d));
  for (int p = 0; p < d; ++p) counts_host[p] = (int64_t)h[p];
  return FTT_OK;
}

int ftt_extract_fibers(ftt_ctx *ctx, const int64_t *coords, const double *values, int64_t nnz,
                       int32_t d, const int64_t *dims_host, int32_t pivot, int64_t *fixed_lin,
                       int64_t *indptr, int64_t *fiber_of, int64_t *pivot_index, double *values_out,
                       int64_t *num_fibers_out) {
  if (!ctx || !num_fibers_out) return FTT_ERR_INVALID;
  FTT_CHECK(check_dims(d, dims_host, pivot, true));
  if (nnz >= ((int64_t)1 << 30)) {
    set_error("nnz exceeds the 2^30 sort limit");
    return FTT_ERR_INVALID;
  }
  if (nnz == 0) {
    *num_fibers_out = 0;
    k_set_i64<<<1, 1, 0, ctx->stream>>>(indptr, 0);
    FTT_LAUNCHED(ctx);
    return FTT_OK;
  }
  FTT_CHECK(arena_reserve(ctx, sort_coords_bytes(nnz, true) + compact_scratch_bytes(nnz) + 1024));
  uint64_t *kr;
  uint32_t *vr;
  uint64_t bound;
  FTT_CHECK(sort_coords(ctx, coords, nnz, d, dims_host, pivot, true, &kr, &vr, &bound));
  int64_t *bc = take<int64_t>(ctx, ceil_div(nnz, CP_TILE) + 1);
  int64_t *total = take<int64_t>(ctx, 1);
  AdjDiffPred pred{kr, make_div63((uint64_t)dims_host[pivot])};
  FiberEmit emit{kr, vr, values, make_div63((uint64_t)dims_host[pivot]), fixed_lin, indptr, fiber_of,
                 pivot_index, values_out};
  // per entry: sorted key + payload + gathered value in; pivot index, value,
  // fiber id out (the per-fiber indptr / key writes are <= 16 bytes x R more)
  FTT_CHECK(compact(ctx, nnz, pred, emit, bc, total, PT_SEGMENT, 44.0 * (double)nnz));
  int64_t R = 0;
  FTT_CHECK(copy_to_host(ctx, &R, total, sizeof(R)));
  k_set_i64<<<1, 1, 0, ctx->stream>>>(indptr + R, nnz);
  FTT_LAUNCHED(ctx);
  *num_fibers_out = R;
  return FTT_OK;
}

// select_p counts from the canonical linear index (see fiber_counts_lin);
// coords (optional) serve the pivots the lin path hands back.
int ftt_fiber_counts_lin(ftt_ctx *ctx, const int64_t *lin, const int64_t *coords, int64_t nnz,
                         int32_t d, const int64_t *dims_host, int64_t *counts_host) {
  if (!ctx || !counts_host || !lin) return FTT_ERR_INVALID;
  FTT_CHECK(check_dims(d, dims_host, 0, false));
  if (nnz >= ((int64_t)1 << 30)) {
    set_error("nnz exceeds the 2^30 sort limit");
    return FTT_ERR_INVALID;
  }
  struct ChunkGuard {  // whatever path runs, no pending lin chunk survives the call
    ftt_ctx *c;
    ~ChunkGuard() { c->lin_nchunks = 0; }
  } chunk_guard{ctx};
  if (nnz == 0) {
    for (int p = 0; p < d; ++p) counts_host[p] = 0;
    return FTT_OK;
  }
  int lg = 1;
  while (((int64_t)1 << lg) < 2 * nnz) ++lg;
  const int64_t T = (int64_t)1 << lg;
  const char *path = getenv("FTT_COUNT_PATH");
  const bool force_lin = path && !strcmp(path, "lin");
  const bool force_other = path && !force_lin;
  if (force_other && coords) {
    FTT_CHECK(lin_chunks_wait_all(ctx));
    return ftt_fiber_counts_all(ctx, coords, nnz, d, dims_host, counts_host);
  }
  if (!force_lin && 8 * T <= ((int64_t)32 << 20)) {
    FTT_CHECK(lin_chunks_wait_all(ctx));
    // small inputs: one pass, d L2-resident global hash sets (as
    // ftt_fiber_counts_all), keys derived from lin
    int group = (int)std::max<int64_t>(1, std::min<int64_t>(d, ((int64_t)1 << 29) / T));
    group = std::min(group, HS_PASS);
    uint64_t *tables = nullptr;
    FTT_CHECK(owned_alloc(ctx, (void **)&tables, 8 * (size_t)T * group + 8 * 32));
    unsigned long long *cnt = reinterpret_cast<unsigned long long *>(tables + (size_t)T * group);
    FTT_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * 32, ctx->stream));
    for (int p0 = 0; p0 < d; p0 += group) {
      const int np = std::min(group, d - p0);
      HashSpec hs;
      hs.d = d;
      hs.np = np;
      hs.lg = lg;
      c_strides(d, dims_host, hs.stride);
      for (int q = 0; q < np; ++q) {
        const uint64_t S = (uint64_t)hs.stride[p0 + q];
        hs.S[q] = S;
        magic_u63(S, &hs.mS[q], &hs.shS[q]);
        magic_u63(S * (uint64_t)dims_host[p0 + q], &hs.mT[q], &hs.shT[q]);
      }
      FTT_CUDA(cudaMemsetAsync(tables, 0xff, 8 * (size_t)T * np, ctx->stream));
      const int pb = prof_begin(ctx);
      k_distinct_hash<<<grid_for(nnz, 256, 1), 256, 0, ctx->stream>>>(
          nullptr, reinterpret_cast<const uint64_t *>(lin), nnz, hs,
          reinterpret_cast<unsigned long long *>(tables), cnt + p0);
      FTT_LAUNCHED(ctx);
      prof_end(ctx, pb, PT_HIST, (double)nnz * (8.0 + 8.0 * np), 0.0);
    }
    unsigned long long h[32];
    FTT_CHECK(copy_to_host(ctx, h, cnt, sizeof(unsigned long long) * d));
    owned_free(ctx, tables);
    for (int p = 0; p < d; ++p) counts_host[p] = (int64_t)h[p];
    return FTT_OK;
  }
  bool done[32];
  FTT_CHECK(fiber_counts_lin(ctx, reinterpret_cast<const uint64_t *>(lin), nnz, d, dims_host,
                             counts_host, done));
  bool all = true;
  for (int p = 0; p < d; ++p) all &= done[p];
  if (all) return FTT_OK;
  static const bool debug = getenv("FTT_DEBUG") != nullptr;
  if (debug)
    for (int p = 0; p < d; ++p)
      if (!done[p]) fprintf(stderr, "[ftt] select_p lin count: pivot %d -> partition\n", p);
  int64_t *cbuf = nullptr;
  if (!coords) {  // the leftovers need coordinates: rebuild them from lin
    FTT_CHECK(owned_alloc(ctx, (void **)&cbuf, 8 * (size_t)nnz * d));
    FTT_CHECK(ftt_delinearize(ctx, lin, nnz, d, dims_host, cbuf));
    coords = cbuf;
  }
  const int rc = fiber_counts_partition(ctx, coords, nnz, d, dims_host, counts_host, done);
  if (cbuf) owned_free(ctx, cbuf);
  return rc;
}

int ftt_extract_fibers_lin(ftt_ctx *ctx, const int64_t *lin, const double *values, int64_t nnz,
                           int32_t d, const int64_t *dims_host, int32_t pivot, int64_t *fixed_lin,
                           int64_t *indptr, int64_t *fiber_of, int64_t *pivot_index,
                           double *values_out, int64_t *num_fibers_out) {
  if (!ctx || !num_fibers_out || !lin) return FTT_ERR_INVALID;
  FTT_CHECK(check_dims(d, dims_host, pivot, true));
  if (nnz >= ((int64_t)1 << 30)) {
    set_error("nnz exceeds the 2^30 sort limit");
    return FTT_ERR_INVALID;
  }
  FTT_CHECK(lin_chunks_wait_all(ctx));
  if (nnz == 0) {
    *num_fibers_out = 0;
    k_set_i64<<<1, 1, 0, ctx->stream>>>(indptr, 0);
    FTT_LAUNCHED(ctx);
    return FTT_OK;
  }
  FTT_CHECK(arena_reserve(ctx, sort_coords_bytes(nnz, true) + compact_scratch_bytes(nnz) + 1024));
  uint64_t *kr;
  uint32_t *vr;
  LinKeySpec ks;
  FTT_CHECK(fiber_keys_lin(ctx, reinterpret_cast<const uint64_t *>(lin), nnz, d, dims_host, pivot,
                           &kr, &vr, &ks));
  int64_t *bc = take<int64_t>(ctx, ceil_div(nnz, CP_TILE) + 1);
  int64_t *total = take<int64_t>(ctx, 1);
  AdjDiffPred pred{kr, make_div63(1)};
  if (ctx->values_event) {  // the values' upload overlapped the key sort (ftt_fasttt_lin)
    FTT_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->values_event, 0));
    ctx->values_event = nullptr;
  }
  FiberEmitLin emit{kr, vr, values, reinterpret_cast<const uint64_t *>(lin), ks, fixed_lin, indptr,
                    fiber_of, pivot_index, values_out};
  FTT_CHECK(compact(ctx, nnz, pred, emit, bc, total, PT_SEGMENT, 44.0 * (double)nnz));
  int64_t R = 0;
  FTT_CHECK(copy_to_host(ctx, &R, total, sizeof(R)));
  k_set_i64<<<1, 1, 0, ctx->stream>>>(indptr + R, nnz);
  FTT_LAUNCHED(ctx);
  *num_fibers_out = R;
  return FTT_OK;
}

int ftt_linearize(ftt_ctx *ctx, const int64_t *coords, int64_t nnz, int32_t d,
                  const int64_t *dims_host, int64_t *lin_out) {
  if (!ctx || (nnz > 0 && (!coords || !lin_out))) return FTT_ERR_INVALID;
  FTT_CHECK(check_dims(d, dims_host, 0, false));
  if (nnz == 0) return FTT_OK;
  LinSpec ls;
  ls.d = d;
  c_strides(d, dims_host, ls.stride);
  k_linearize_c<<<grid_for(nnz, 256, 4), 256, 0, ctx->stream>>>(coords, nnz, ls, lin_out);
  FTT_LAUNCHED(ctx);
  return FTT_OK;
}

static int depar_from_keys(ftt_ctx *ctx, int64_t n_rows, int64_t R, const SweepKey *skey,
                           const int64_t *rows, int64_t *kept, int64_t *map_out,
                           int64_t *n_kept_out) {
  // rows (explicit col_to_row) or skey (computed) gives key(f) for f < R
  const bool flag_path = n_rows <= ((int64_t)1 << 31) - 1 &&
                         (n_rows <= ((int64_t)1 << 24) || n_rows <= 8 * R);
  if (flag_path) {
    FTT_CHECK(arena_reserve(ctx, align_up(4 * n_rows) + compact_scratch_bytes(n_rows) + 1024));
    uint32_t *present = take<uint32_t>(ctx, n_rows);
    int64_t *bc = take<int64_t>(ctx, ceil_div(n_rows, CP_TILE) + 1);
    int64_t *total = take<int64_t>(ctx, 1);
    FTT_CUDA(cudaMemsetAsync(present, 0, 4 * n_rows, ctx->stream));
    const int pb = prof_begin(ctx);
    if (skey) {
      k_sweep_mark<<<grid_for(R, 256, 4), 256, 0, ctx->stream>>>(R, *skey, present);
    } else {
      k_mark_rows<<<grid_for(R, 256, 4), 256, 0, ctx->stream>>>(R, rows, present);
    }
    FTT_LAUNCHED(ctx);
    FTT_CHECK(compact(ctx, n_rows, FlagPred{present}, KeptEmit{present, kept}, bc, total, -1));
    if (skey) {
      k_sweep_gather<<<grid_for(R, 256, 4), 256, 0, ctx->stream>>>(R, *skey, present, map_out);
    } else {
      k_gather_rank<<<grid_for(R, 256, 4), 256, 0, ctx->stream>>>(R, rows, present, map_out);
    }
    FTT_LAUNCHED(ctx);
    // mark: key inputs (16 B) per fiber + flag write; scan: flags; gather:
    // key inputs again + rank read + map write (kept writes <= 8 B x R)
    prof_end(ctx, pb, PT_SWEEP, (double)R * (16.0 + 4.0 + 16.0 + 4.0 + 8.0) + 8.0 * (double)n_rows,
             0.0);
    FTT_CHECK(copy_to_host(ctx, n_kept_out, total, sizeof(int64_t)));
    return FTT_OK;
  }
  // sort path: unique over R keys
  if (R >= ((int64_t)1 << 30)) {
    set_error("fiber count exceeds the 2^30 sort limit");
    return FTT_ERR_INVALID;
  }
  FTT_CHECK(arena_reserve(ctx, radix_sort_scratch_bytes(R, true) + 2 * align_up(8 * R) +
                                   2 * align_up(4 * R) + compact_scratch_bytes(R) + 1024));
  uint64_t *keys = take<uint64_t>(ctx, R);
  uint64_t *skeys = take<uint64_t>(ctx, R);
  uint32_t *perm = take<uint32_t>(ctx, R);
  int64_t *bc = take<int64_t>(ctx, ceil_div(R, CP_TILE) + 1);
  int64_t *total = take<int64_t>(ctx, 1);
  if (skey) {
    k_sweep_keys<<<grid_for(R, 256, 4), 256, 0, ctx->stream>>>(R, *skey, keys);
  } else {
    k_copy_keys<<<grid_for(R, 256, 4), 256, 0, ctx->stream>>>(R, rows, keys);
  }
  FTT_LAUNCHED(ctx);
  // identity payload is produced by the histogram kernel inside radix_sort
  // only for coords; build it here explicitly.
  uint32_t *ident = take<uint32_t>(ctx, R);
  if (!ident) {
    set_error("depar: arena too small");
    return FTT_ERR_INVALID;
  }
  {
    // reuse k_hist's idx output to fill the identity permutation
    uint32_t *dummy_hist = take<uint32_t>(ctx, 8 * RADIX);
    FTT_CUDA(cudaMemsetAsync(dummy_hist, 0, sizeof(uint32_t) * 8 * RADIX, ctx->stream));
    k_hist<<<grid_for(R, 256, 8), 256, 0, ctx->stream>>>(keys, R, 0, dummy_hist, ident);
    FTT_LAUNCHED(ctx);
  }
  FTT_CHECK(radix_sort(ctx, keys, ident, skeys, perm, R, bit_length((uint64_t)(n_rows - 1))));
  FTT_CHECK(compact(ctx, R, AdjDiffPred{skeys, make_div63(1)}, UniqEmit{skeys, perm, kept, map_out}, bc, total));
  FTT_CHECK(copy_to_host(ctx, n_kept_out, total, sizeof(int64_t)));
  return FTT_OK;
}

int ftt_depar_quasi_perm(ftt_ctx *ctx, int64_t n_rows, int64_t n_cols, const int64_t *col_to_row,
                         int64_t *kept, int64_t *t_map, int64_t *n_kept_out) {
  if (!ctx || !n_kept_out || n_rows < 0 || n_cols < 0) return FTT_ERR_INVALID;
  if (n_cols == 0 || n_rows == 0) {
    *n_kept_out = 0;
    return FTT_OK;
  }
  return depar_from_keys(ctx, n_rows, n_cols, nullptr, col_to_row, kept, t_map, n_kept_out);
}

int ftt_index_sweep_step(ftt_ctx *ctx, int32_t side, const int64_t *fixed_lin, int64_t R,
                         int64_t stride_k, int64_t n_k, const int64_t *map_in, int64_t r_other,
                         int64_t *kept, int64_t *map_out, int64_t *n_kept_out) {
  if (!ctx || !n_kept_out || (side != 0 && side != 1) || stride_k < 1 || n_k < 1 || r_other < 1) {
    set_error("ftt_index_sweep_step: invalid arguments");
    return FTT_ERR_INVALID;
  }
  if (R == 0) {
    *n_kept_out = 0;
    return FTT_OK;
  }
  SweepKey sk{side, fixed_lin, stride_k, n_k, r_other, map_in, make_div63((uint64_t)stride_k),
              make_div63((uint64_t)n_k)};
  return depar_from_keys(ctx, r_other * n_k, R, &sk, nullptr, kept, map_out, n_kept_out);
}

// All deparallelisation steps of _index_sweeps (fasttt.py:181-211) in one
// call with one host round trip: each step's kept count stays on the device
// and feeds the next step's key (right side: i_k * r_next + s_map) directly.
// The flag array is sized by a host-side bound of r_other * n_k (min(R,
// product of the dims already swept)) and cleaned after each step by
// unmarking the step's kept rows, so no per-step memset or count read-back
// is needed.  Returns FTT_ERR_INVALID (nothing launched) when a bound is too
// large for the flag path -- the caller then runs ftt_index_sweep_step per
// step.  kept[s] / maps[s] (step s: left k = 0..p-1, then right k =
// d-1..p+1) hold min(R, bound_s) / R entries; n_kept_out[s] gets the counts.
int ftt_index_sweeps_all(ftt_ctx *ctx, const int64_t *fixed_lin, int64_t R, int32_t d,
                         const int64_t *dims, int32_t pivot, int64_t *const *kept,
                         int64_t *const *maps, int64_t *n_kept_out) {
  if (!ctx || !n_kept_out || d < 2 || d > 32 || pivot < 0 || pivot >= d || R < 1) {
    set_error("ftt_index_sweeps_all: invalid arguments");
    return FTT_ERR_INVALID;
  }
  const int nsteps = d - 1;
  std::vector<int64_t> bound(nsteps), nk(nsteps), stride(nsteps);
  std::vector<int> side(nsteps);
  {
    // rest strides: C order over the modes != pivot
    std::vector<int64_t> rest_stride(d, 0);
    int64_t st = 1;
    for (int k = d - 1; k >= 0; --k) {
      if (k == pivot) continue;
      rest_stride[k] = st;
      st *= dims[k];
    }
    int s = 0;
    int64_t prod = 1;
    for (int k = 0; k < pivot; ++k, ++s) {
      side[s] = 0;
      nk[s] = dims[k];
      stride[s] = rest_stride[k];
      bound[s] = std::min<int64_t>(R, prod) * dims[k];
      prod = std::min<int64_t>(prod * dims[k], (int64_t)1 << 40);
    }
    prod = 1;
    for (int k = d - 1; k > pivot; --k, ++s) {
      side[s] = 1;
      nk[s] = dims[k];
      stride[s] = rest_stride[k];
      bound[s] = std::min<int64_t>(R, prod) * dims[k];
      prod = std::min<int64_t>(prod * dims[k], (int64_t)1 << 40);
    }
  }
  // flag rows per step: r_other * n_k with r_other the previous step's count
  // (read on the device: no host round trip between steps); the flag array
  // is the context's persistent zeroed one, sized for the static bound
  int64_t bmax = 1;
  for (int s = 0; s < nsteps; ++s) {
    if (bound[s] > ((int64_t)1 << 31) - 1) {
      set_error("ftt_index_sweeps_all: flag bound too large");
      return FTT_ERR_INVALID;
    }
    bmax = std::max(bmax, bound[s]);
  }
  // two zeroed flag arrays: step s ranks in flags[s & 1] while marking step
  // s + 1's keys in the other (fused gather + mark)
  uint32_t *zf = nullptr;
  FTT_CHECK(zero_flags(ctx, 2 * (size_t)bmax, &zf));
  uint32_t *flags[2] = {zf, zf + bmax};
  FTT_CHECK(arena_reserve(ctx, compact_scratch_bytes(bmax) + align_up(8 * (size_t)(nsteps + 1)) +
                                   4096));
  int64_t *bc = take<int64_t>(ctx, ceil_div(bmax, CP_TILE) + 1);
  int64_t *counts = take<int64_t>(ctx, nsteps + 1);
  const int pb = prof_begin(ctx);
  double alg = 0.0;
  auto key_of = [&](int st) {
    // previous step of the same side: its map and its count
    const bool first = (st == 0) || side[st - 1] != side[st];
    SweepKey sk{side[st], fixed_lin, stride[st], nk[st], 1, first ? nullptr : maps[st - 1],
                make_div63((uint64_t)stride[st]), make_div63((uint64_t)nk[st])};
    if (side[st] == 1 && !first) sk.r_other_dev = counts + (st - 1);
    return sk;
  };
  k_sweep_mark<<<grid_for(R, 256, 4), 256, 0, ctx->stream>>>(R, key_of(0), flags[0]);
  FTT_LAUNCHED(ctx);
  for (int s = 0; s < nsteps; ++s) {
    const bool first_of_side = (s == 0) || side[s - 1] != side[s];
    const SweepKey sk = key_of(s);
    uint32_t *present = flags[s & 1];
    const int64_t *ndev = first_of_side ? nullptr : counts + (s - 1);
    const int64_t nrows = first_of_side ? nk[s] : bound[s];
    FTT_CHECK(compact(ctx, nrows, FlagPred{present}, KeptEmit{present, kept[s]}, bc, counts + s, -1,
                      0.0, ndev, nk[s]));
    if (s + 1 < nsteps) {
      const bool next_first = side[s + 1] != side[s];
      k_sweep_gather_mark<<<grid_for(R, 256, 4), 256, 0, ctx->stream>>>(
          R, sk, present, maps[s], key_of(s + 1), next_first ? 0 : 1, flags[(s + 1) & 1]);
    } else {
      k_sweep_gather<<<grid_for(R, 256, 4), 256, 0, ctx->stream>>>(R, sk, present, maps[s]);
    }
    FTT_LAUNCHED(ctx);
    k_unmark<<<grid_for(std::min(R, bound[s]), 256, 4), 256, 0, ctx->stream>>>(
        kept[s], counts + s, std::min(R, bound[s]), present);
    FTT_LAUNCHED(ctx);
    alg += (double)R * (16.0 + 4.0 + 8.0 + 4.0);
  }
  prof_end(ctx, pb, PT_SWEEP, alg, 0.0);
  FTT_CHECK(copy_to_host(ctx, n_kept_out, counts, sizeof(int64_t) * nsteps));
  return FTT_OK;
}

int ftt_mode_index(ftt_ctx *ctx, const int64_t *fixed_lin, int64_t R, int64_t stride, int64_t n,
                   int64_t *out) {
  if (!ctx || stride < 1 || n < 1) return FTT_ERR_INVALID;
  if (R == 0) return FTT_OK;
  k_mode_index<<<grid_for(R, 256, 4), 256, 0, ctx->stream>>>(fixed_lin, R, stride, n, out);
  FTT_LAUNCHED(ctx);
  return FTT_OK;
}

int ftt_pivot_core_scatter(ftt_ctx *ctx, int64_t nnz, const int64_t *fiber_of,
                           const int64_t *pivot_index, const double *values, const int64_t *t_map,
                           const int64_t *s_map, int64_t r_prev, int64_t n_p, int64_t r_next,
                           double *core, double *norm_out) {
  if (!ctx) return FTT_ERR_INVALID;
  size_t elems = (size_t)r_prev * n_p * r_next;
  FTT_CUDA(cudaMemsetAsync(core, 0, elems * sizeof(double), ctx->stream));
  int nb = grid_for(nnz, 256, 4, 148 * 8);
  FTT_CHECK(arena_reserve(ctx, align_up(8 * (nb + 1)) + 256));
  double *partial = take<double>(ctx, nb + 1);
  if (nnz > 0) {
    const int pb = prof_begin(ctx);
    k_pivot_scatter<<<nb, 256, 0, ctx->stream>>>(nnz, fiber_of, pivot_index, values, t_map, s_map,
                                                 n_p, r_next, core, partial);
    FTT_LAUNCHED(ctx);
    // fiber id, pivot index, value, two map reads and the scattered write
    prof_end(ctx, pb, PT_SCATTER, 48.0 * (double)nnz, 0.0);
  }
  if (norm_out) {
    if (nnz == 0) {
      *norm_out = 0.0;
      return FTT_OK;
    }
    k_reduce_partials<<<1, 1024, 0, ctx->stream>>>(partial, nb, partial + nb);
    FTT_LAUNCHED(ctx);
    double s2 = 0;
    FTT_CHECK(copy_to_host(ctx, &s2, partial + nb, sizeof(double)));
    *norm_out = sqrt(s2);
  }
  return FTT_OK;
}

int ftt_side_core_dense(ftt_ctx *ctx, int32_t side, const int64_t *kept, int64_t K, int64_t n,
                        int64_t r_other, double *core) {
  if (!ctx || (side != 0 && side != 1)) return FTT_ERR_INVALID;
  FTT_CUDA(cudaMemsetAsync(core, 0, sizeof(double) * (size_t)K * n * r_other, ctx->stream));
  if (K > 0) {
    k_side_core<<<grid_for(K, 256, 4), 256, 0, ctx->stream>>>(side, kept, K, n, r_other, core);
    FTT_LAUNCHED(ctx);
  }
  return FTT_OK;
}

int ftt_scatter_cols(ftt_ctx *ctx, int64_t rank, int64_t K, const int64_t *kept, const double *src,
                     int64_t lds, int64_t ncols_new, double *dst) {
  if (!ctx) return FTT_ERR_INVALID;
  FTT_CUDA(cudaMemsetAsync(dst, 0, sizeof(double) * (size_t)rank * ncols_new, ctx->stream));
  if (rank * K > 0) {
    k_scatter_cols<<<grid_for(rank * K, 256, 4), 256, 0, ctx->stream>>>(rank, K, kept, src, lds,
                                                                       ncols_new, dst);
    FTT_LAUNCHED(ctx);
  }
  return FTT_OK;
}

int ftt_scatter_rows(ftt_ctx *ctx, int64_t K, int64_t rank, const int64_t *kept, const double *src,
                     int64_t lds, int64_t nrows_new, double *dst) {
  if (!ctx) return FTT_ERR_INVALID;
  FTT_CUDA(cudaMemsetAsync(dst, 0, sizeof(double) * (size_t)nrows_new * rank, ctx->stream));
  if (rank * K > 0) {
    k_scatter_rows<<<grid_for(rank * K, 256, 4), 256, 0, ctx->stream>>>(K, rank, kept, src, lds,
                                                                       dst);
    FTT_LAUNCHED(ctx);
  }
  return FTT_OK;
}

int ftt_dot(ftt_ctx *ctx, int64_t n, const double *x, const double *y, double *out_host) {
  if (!ctx || !out_host) return FTT_ERR_INVALID;
  if (n == 0) {
    *out_host = 0.0;
    return FTT_OK;
  }
  int nb = grid_for(n, 256, 4, 148 * 8);
  FTT_CHECK(arena_reserve(ctx, align_up(8 * (nb + 1)) + 256));
  double *partial = take<double>(ctx, nb + 1);
  k_dot_partial<<<nb, 256, 0, ctx->stream>>>(n, x, y, partial, partial + nb,
                                             ctx->tile_cnt + kTileCnt);
  FTT_LAUNCHED(ctx);
  return copy_to_host(ctx, out_host, partial + nb, sizeof(double));
}


int ftt_tensorize_matrix(ftt_ctx *ctx, int64_t nnz, const int64_t *rows, const int64_t *cols,
                         const double *vals, int32_t d, const int64_t *row_dims,
                         const int64_t *col_dims, int64_t *coords_out, double *vals_out,
                         int64_t *nnz_out) {
  if (!ctx || !nnz_out || d < 1 || d > 32 || nnz < 0) {
    set_error("ftt_tensorize_matrix: invalid arguments");
    return FTT_ERR_INVALID;
  }
  FuseSpec fs;
  fs.d = d;
  int64_t fused[32];
  for (int i = 0; i < d; ++i) {
    fs.rdims[i] = row_dims[i];
    fs.cdims[i] = col_dims[i];
    fused[i] = row_dims[i] * col_dims[i];
  }
  FTT_CHECK(check_dims(d, fused, 0, false));
  unsigned __int128 prod = 1;
  for (int i = d - 1; i >= 0; --i) {
    fs.stride[i] = (int64_t)prod;
    prod *= (unsigned __int128)fused[i];
  }
  *nnz_out = 0;
  if (nnz == 0) return FTT_OK;
  if (nnz >= ((int64_t)1 << 30)) {
    set_error("nnz exceeds the 2^30 sort limit");
    return FTT_ERR_INVALID;
  }
  FTT_CHECK(arena_reserve(ctx, radix_sort_scratch_bytes(nnz, true) + 2 * align_up(8 * nnz) +
                                   2 * align_up(4 * nnz) + compact_scratch_bytes(nnz) + 4096));
  uint64_t *keys = take<uint64_t>(ctx, nnz), *skeys = take<uint64_t>(ctx, nnz);
  uint32_t *ident = take<uint32_t>(ctx, nnz), *perm = take<uint32_t>(ctx, nnz);
  int64_t *bc = take<int64_t>(ctx, ceil_div(nnz, CP_TILE) + 1);
  int64_t *total = take<int64_t>(ctx, 2);  // [0] kept entries, [1] out-of-range flag
  int *bad = reinterpret_cast<int *>(total + 1);
  FTT_CUDA(cudaMemsetAsync(total + 1, 0, sizeof(int64_t), ctx->stream));
  k_fuse_keys<<<grid_for(nnz, 256, 4), 256, 0, ctx->stream>>>(nnz, rows, cols, fs, keys, ident, bad);
  FTT_LAUNCHED(ctx);
  FTT_CHECK(radix_sort(ctx, keys, ident, skeys, perm, nnz, bit_length((uint64_t)(prod - 1))));
  CoalescePred pred{skeys, perm, vals, nnz};
  FTT_CHECK(compact(ctx, nnz, pred, CoalesceEmit{pred, fs, coords_out, vals_out}, bc, total));
  int64_t h[2] = {0, 0};
  FTT_CHECK(copy_to_host(ctx, h, total, 2 * sizeof(int64_t)));
  if ((int)h[1]) {
    set_error("matrix entry outside the factored extents");
    return FTT_ERR_INVALID;
  }
  *nnz_out = h[0];
  return FTT_OK;
}


int ftt_delinearize(ftt_ctx *ctx, const int64_t *lin, int64_t nnz, int32_t d,
                    const int64_t *dims_host, int64_t *coords_out) {
  if (!ctx || d < 1 || d > 32 || nnz < 0) {
    set_error("ftt_delinearize: invalid arguments");
    return FTT_ERR_INVALID;
  }
  FTT_CHECK(check_dims(d, dims_host, 0, false));
  if (nnz == 0) return FTT_OK;
  DelinSpec ds;
  ds.d = d;
  int64_t st = 1;
  for (int k = d - 1; k >= 0; --k) {
    ds.stride[k] = st;
    st *= dims_host[k];
  }
  for (int k = 0; k < d; ++k) magic_u63((uint64_t)ds.stride[k], &ds.m[k], &ds.sh[k]);
  const int pb = prof_begin(ctx);
  k_delinearize<<<grid_for(nnz, 256, 4), 256, 0, ctx->stream>>>(lin, nnz, ds, coords_out);
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb, PT_HIST, (double)nnz * (8.0 + 8.0 * d), 0.0);
  return FTT_OK;
}

}  // extern "C"
