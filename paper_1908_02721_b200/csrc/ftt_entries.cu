// tt_entries (ttformat.py:124-136): entries of a train at many coordinates.
// Used by the error report of fasttt (sparse_inner_error, fasttt.py:587-602)
// and by the parity checks.
//  * max rank <= 64: one warp per coordinate, the running row vector lives
//    in two registers per lane, slices are read coalesced along r_{k+1}.
//  * larger ranks: level-by-level grouped GEMMs -- rows are stably sorted by
//    the mode-k index so that every group shares one (r_k x r_{k+1}) slice,
//    which turns the per-coordinate GEMVs into DMMA GEMMs.
#include <algorithm>
#include <vector>

#include "ftt_dense.cuh"

namespace ftt {
namespace {

struct TrainDesc {
  int d;
  int64_t dims[32];
  int64_t ranks[33];
  const double *cores[32];
};

__global__ void k_entries_small(TrainDesc t, const int64_t *__restrict__ coords, int64_t n,
                                double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    double v0 = lane == 0 ? 1.0 : 0.0, v1 = 0.0;
    for (int k = 0; k < t.d; ++k) {
      const int64_t r0 = t.ranks[k], r1 = t.ranks[k + 1], nk = t.dims[k];
      const int64_t idx = coords[i * t.d + k];
      const double *G = t.cores[k] + idx * r1;
      const int64_t rowst = nk * r1;
      double a0 = 0.0, a1 = 0.0;
      for (int64_t a = 0; a < r0; ++a) {
        double va = __shfl_sync(0xffffffffu, a < 32 ? v0 : v1, (int)(a & 31));
        if (lane < r1) a0 += va * G[a * rowst + lane];
        if (lane + 32 < r1) a1 += va * G[a * rowst + lane + 32];
      }
      v0 = a0;
      v1 = a1;
    }
    if (lane == 0) out[i] = v0;
  }
}

// Ranks <= L (L = 4, 8, 16, 32): a group of L lanes per coordinate (32 / L
// coordinates per warp), the running row vector one register per lane,
// broadcasts by width-L shuffles.  Latency hiding: the point's coordinates
// are loaded once up front (lane s of the group holds modes s, s + L, ...),
// and the core slice of step k + 1 is loaded before the FMAs of step k.
template <int L>
__device__ __forceinline__ void load_slice(const TrainDesc &t, int k, int64_t idx, int sub, bool act,
                                           double (&g)[L]) {
  const int r0 = (int)t.ranks[k], r1 = (int)t.ranks[k + 1];
  const int rowst = (int)t.dims[k] * r1;  // < 2^31 for the ranks <= 32 of this path
  const double *G = t.cores[k] + (idx * r1 + sub);
  const bool on = act && sub < r1;
#pragma unroll
  for (int a = 0; a < L; ++a) {
    g[a] = (on && a < r0) ? __ldg(G) : 0.0;
    G += rowst;
  }
}

template <int L>
__global__ void __launch_bounds__(256) k_entries_grp(TrainDesc t, const int64_t *__restrict__ coords,
                                                     int64_t n, double *__restrict__ out) {
  constexpr int CW = (32 + L - 1) / L;  // coordinate registers per lane (d <= 32)
  const int lane = threadIdx.x & 31, sub = lane & (L - 1);
  constexpr int PER_WARP = 32 / L;
  const int64_t slots = (int64_t)gridDim.x * (blockDim.x >> 5) * PER_WARP;
  const int64_t first = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * PER_WARP +
                        (lane / L);
  // every lane of a warp runs the same trip count (shuffles need the full warp)
  const int64_t trips = (n + slots - 1) / slots;
  const int d = t.d;
  for (int64_t it = 0; it < trips; ++it) {
    const int64_t i = first + it * slots;
    const bool live = i < n;
    int64_t cw[CW];
#pragma unroll
    for (int u = 0; u < CW; ++u) {
      const int k = sub + u * L;
      cw[u] = (live && k < d) ? coords[i * d + k] : 0;
    }
    auto coord = [&](int k) -> int64_t {  // mode-k index of this group's point
      int64_t x = cw[0];
#pragma unroll
      for (int u = 1; u < CW; ++u)
        if (k / L == u) x = cw[u];
      return __shfl_sync(0xffffffffu, x, k & (L - 1), L);
    };
    double v = sub == 0 ? 1.0 : 0.0;
    double g[L], gn[L];
    load_slice<L>(t, 0, coord(0), sub, live, g);
    for (int k = 0; k < d; ++k) {
      if (k + 1 < d) load_slice<L>(t, k + 1, coord(k + 1), sub, live, gn);
      const int r0 = (int)t.ranks[k];
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < L; ++a) {
        const double va = __shfl_sync(0xffffffffu, v, a, L);
        if (a < r0) acc += va * g[a];
      }
      v = acc;
#pragma unroll
      for (int a = 0; a < L; ++a) g[a] = gn[a];
    }
    if (live && sub == 0) out[i] = v;
  }
}

// Ranks <= R (4 / 8): one thread per coordinate, the running row vector in
// R registers; each core slice row is read as double2 pairs (rows of r_{k+1}
// contiguous doubles).  ~20 warp instructions per coordinate for config 2
// (ranks 8) against ~10x that for the lane-group kernel; consecutive
// coordinates share their leading modes (C-sorted input), so the slice
// loads of those modes are broadcast within a warp.
template <int R>
__global__ void __launch_bounds__(256) k_entries_thr(TrainDesc t, const int64_t *__restrict__ coords,
                                                     int64_t n, double *__restrict__ out,
                                                     int aligned16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v[R];
#pragma unroll
    for (int a = 0; a < R; ++a) v[a] = a == 0 ? 1.0 : 0.0;
    const int64_t *c = coords + i * t.d;
    for (int k = 0; k < t.d; ++k) {
      const int r0 = (int)t.ranks[k], r1 = (int)t.ranks[k + 1];
      const int64_t rowst = t.dims[k] * r1;
      const double *G = t.cores[k] + c[k] * r1;
      double acc[R];
#pragma unroll
      for (int b = 0; b < R; ++b) acc[b] = 0.0;
      if ((r1 & 1) == 0 && aligned16) {
#pragma unroll
        for (int a = 0; a < R; ++a) {
          if (a < r0) {
            const double2 *row = reinterpret_cast<const double2 *>(G + a * rowst);
#pragma unroll
            for (int b = 0; b < R; b += 2)
              if (b < r1) {
                const double2 g = __ldg(row + b / 2);
                acc[b] += v[a] * g.x;
                acc[b + 1] += v[a] * g.y;
              }
          }
        }
      } else {
#pragma unroll
        for (int a = 0; a < R; ++a)
          if (a < r0) {
            const double *row = G + a * rowst;
#pragma unroll
            for (int b = 0; b < R; ++b)
              if (b < r1) acc[b] += v[a] * __ldg(row + b);
          }
      }
#pragma unroll
      for (int b = 0; b < R; ++b) v[b] = acc[b];
    }
    out[i] = v[0];
  }
}

__global__ void k_first_rows(int64_t n, const int64_t *__restrict__ coords, int d, const double *core0,
                             int64_t r1, const int64_t *__restrict__ idx, double *__restrict__ V) {
  int64_t total = n * r1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / r1, j = t - i * r1;
    V[t] = core0[coords[idx[i] * d] * r1 + j];
  }
}

__global__ void k_level_keys(int64_t n, const int64_t *__restrict__ coords, int d, int k,
                             const int64_t *__restrict__ idx, uint64_t *__restrict__ keys,
                             uint32_t *__restrict__ pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = (uint64_t)coords[idx[i] * d + k];
    pos[i] = (uint32_t)i;
  }
}

__global__ void k_permute_rows(int64_t n, int64_t r, const uint32_t *__restrict__ perm,
                               const double *__restrict__ V, double *__restrict__ Vs,
                               const int64_t *__restrict__ idx, int64_t *__restrict__ idx_new) {
  int64_t total = n * r;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / r, j = t - i * r;
    int64_t src = perm[i];
    Vs[t] = V[src * r + j];
    if (j == 0) idx_new[i] = idx[src];
  }
}

__global__ void k_bounds(int64_t n, const uint64_t *__restrict__ skeys, int64_t nk, int64_t *__restrict__ off) {
  // off[v] = first position with key >= v (sorted keys), off[nk] = n
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = i == 0 ? 0 : (int64_t)skeys[i - 1] + 1;
    int64_t hi = i == n ? nk : (int64_t)skeys[i];
    for (int64_t v = lo; v <= hi && v <= nk; ++v) off[v] = i;
  }
}

__global__ void k_scatter_out(int64_t n, int64_t r, const double *__restrict__ V,
                              const int64_t *__restrict__ idx, double *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[idx[i]] = V[i * r];
}

__global__ void k_iota64(int64_t n, int64_t base, int64_t *p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = base + i;
}

// ---------------------------------------------------------------- meet in
// the middle (ranks <= 64): entry(i) = L[prefix(i)] . R[suffix(i)] where L
// (R) chains the cores left (right) of the split for each DISTINCT prefix
// (suffix) only.  Sorted COO input shares prefixes heavily (config 5:
// 8.5M nonzeros, 11,664 distinct 6-mode prefixes), so the per-nonzero work
// drops from d r^2 MACs to r.
constexpr int MT_TILE = 4096;

__global__ void k_half_keys(int64_t n, const int64_t *__restrict__ coords, int d, int k0, int k1,
                            TrainDesc t, uint64_t *__restrict__ keys, uint32_t *__restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t key = 0;
    for (int k = k0; k < k1; ++k) key = key * (uint64_t)t.dims[k] + (uint64_t)coords[i * d + k];
    keys[i] = key;
    idx[i] = (uint32_t)i;
  }
}

__global__ void k_seg_count(int64_t n, const uint64_t *__restrict__ k, int64_t *__restrict__ bc) {
  __shared__ int s[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * MT_TILE;
  int c = 0;
  for (int64_t i = base + threadIdx.x; i < min(n, base + MT_TILE); i += 256)
    c += (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
  for (int off = 16; off; off >>= 1) c += __shfl_down_sync(0xffffffffu, c, off);
  if (lane == 0) s[warp] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t tsum = 0;
    for (int w = 0; w < 8; ++w) tsum += s[w];
    bc[blockIdx.x] = tsum;
  }
}

// ids_of[payload[i]] = id of sorted key i; uniq[id] = key at its first position
__global__ void k_seg_assign(int64_t n, const uint64_t *__restrict__ k,
                             const uint32_t *__restrict__ payload, const int64_t *__restrict__ off,
                             int64_t *__restrict__ ids_of, uint64_t *__restrict__ uniq) {
  __shared__ int s[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * MT_TILE;
  // warp-contiguous chunks of 512, processed in 16 rounds of 32
  const int64_t wbase = base + warp * 512;
  int cnt = 0;
  unsigned balls[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    int64_t i = wbase + j * 32 + lane;
    bool f = i < n && (i == 0 || k[i] != k[i - 1]);
    balls[j] = __ballot_sync(0xffffffffu, f);
    cnt += __popc(balls[j]);
  }
  if (lane == 0) s[warp] = cnt;
  __syncthreads();
  int64_t run = off[blockIdx.x];
  for (int w = 0; w < warp; ++w) run += s[w];
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    int64_t i = wbase + j * 32 + lane;
    bool f = (balls[j] >> lane) & 1u;
    int64_t id = run + __popc(balls[j] & lt) + (f ? 0 : -1);
    if (i < n) {
      ids_of[payload[i]] = id;
      if (f) uniq[id] = k[i];
    }
    run += __popc(balls[j]);
  }
}

// One warp per distinct half-key: the chained row (left, from core k0) or
// column (right, from core k1-1 backwards) vector of the cores [k0, k1).
__global__ void k_half_vectors(int64_t nk, const uint64_t *__restrict__ uniq, TrainDesc t, int k0,
                               int k1, int left, double *__restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); u < nk; u += warps) {
    uint64_t key = uniq[u];
    int64_t idx[32];
    for (int k = k1 - 1; k >= k0; --k) {
      idx[k] = (int64_t)(key % (uint64_t)t.dims[k]);
      key /= (uint64_t)t.dims[k];
    }
    double v0 = lane == 0 ? 1.0 : 0.0, v1 = 0.0;
    if (left) {
      for (int k = k0; k < k1; ++k) {  // v (1 x r_k) <- v @ G_k[:, i_k, :]
        const int64_t r0 = t.ranks[k], r1 = t.ranks[k + 1], nkk = t.dims[k];
        const double *G = t.cores[k] + idx[k] * r1;
        double a0 = 0.0, a1 = 0.0;
        for (int64_t a = 0; a < r0; ++a) {
          double va = __shfl_sync(0xffffffffu, a < 32 ? v0 : v1, (int)(a & 31));
          if (lane < r1) a0 += va * G[a * nkk * r1 + lane];
          if (lane + 32 < r1) a1 += va * G[a * nkk * r1 + lane + 32];
        }
        v0 = a0;
        v1 = a1;
      }
    } else {
      for (int k = k1 - 1; k >= k0; --k) {  // w (r_k x 1) <- G_k[:, i_k, :] @ w
        const int64_t r0 = t.ranks[k], r1 = t.ranks[k + 1], nkk = t.dims[k];
        const double *G = t.cores[k] + idx[k] * r1;
        double a0 = 0.0, a1 = 0.0;
        for (int64_t b = 0; b < r1; ++b) {
          double wb = __shfl_sync(0xffffffffu, b < 32 ? v0 : v1, (int)(b & 31));
          if (lane < r0) a0 += G[(int64_t)lane * nkk * r1 + b] * wb;
          if (lane + 32 < r0) a1 += G[(int64_t)(lane + 32) * nkk * r1 + b] * wb;
        }
        v0 = a0;
        v1 = a1;
      }
    }
    const int64_t rm = left ? t.ranks[k1] : t.ranks[k0];
    if (lane < rm) out[u * ldo + lane] = v0;
    if (lane + 32 < rm) out[u * ldo + lane + 32] = v1;
  }
}

__global__ void k_mitm_dot(int64_t n, int64_t rm, const int64_t *__restrict__ lid,
                           const int64_t *__restrict__ rid, const double *__restrict__ L,
                           const double *__restrict__ R, double *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double *l = L + lid[i] * rm;
    const double *r = R + rid[i] * rm;
    double s = 0.0;
    for (int64_t a = 0; a < rm; ++a) s += l[a] * r[a];
    out[i] = s;
  }
}

int bitlen(uint64_t x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

int entries_mitm(ftt_ctx *ctx, const TrainDesc &t, const int64_t *coords, int64_t n, double *out) {
  const int d = t.d, m = d / 2;
  uint64_t pb = 1, sb = 1;
  for (int k = 0; k < m; ++k) pb *= (uint64_t)t.dims[k];
  for (int k = m; k < d; ++k) sb *= (uint64_t)t.dims[k];
  const int pbits = std::max(1, bitlen(pb - 1)), sbits = std::max(1, bitlen(sb - 1));
  const int64_t rm = t.ranks[m];
  const int64_t nt = ceil_div(n, MT_TILE);
  uint64_t *keys = nullptr, *skeys = nullptr, *uniq[2] = {nullptr, nullptr};
  uint32_t *idx = nullptr, *perm = nullptr;
  int64_t *ids[2] = {nullptr, nullptr}, *bc = nullptr;
  double *vec[2] = {nullptr, nullptr};
  FTT_CHECK(owned_alloc(ctx, (void **)&keys, 8 * (size_t)n));
  FTT_CHECK(owned_alloc(ctx, (void **)&skeys, 8 * (size_t)n));
  FTT_CHECK(owned_alloc(ctx, (void **)&idx, 4 * (size_t)n));
  FTT_CHECK(owned_alloc(ctx, (void **)&perm, 4 * (size_t)n));
  FTT_CHECK(owned_alloc(ctx, (void **)&bc, 8 * (size_t)(nt + 2)));
  int64_t nuniq[2] = {0, 0};
  for (int side = 0; side < 2; ++side) {
    const int k0 = side == 0 ? 0 : m, k1 = side == 0 ? m : d;
    FTT_CHECK(owned_alloc(ctx, (void **)&ids[side], 8 * (size_t)n));
    FTT_CHECK(owned_alloc(ctx, (void **)&uniq[side], 8 * (size_t)n));
    k_half_keys<<<grid_for(n, 256, 4), 256, 0, ctx->stream>>>(n, coords, d, k0, k1, t, keys, idx);
    FTT_LAUNCHED(ctx);
    FTT_CHECK(arena_reserve(ctx, radix_sort_scratch_bytes(n, true) + 1024));
    FTT_CHECK(radix_sort(ctx, keys, idx, skeys, perm, n, side == 0 ? pbits : sbits));
    k_seg_count<<<(unsigned)nt, 256, 0, ctx->stream>>>(n, skeys, bc);
    FTT_LAUNCHED(ctx);
    FTT_CHECK(scan_block_counts(ctx, bc, nt, bc + nt + 1));
    k_seg_assign<<<(unsigned)nt, 256, 0, ctx->stream>>>(n, skeys, perm, bc, ids[side], uniq[side]);
    FTT_LAUNCHED(ctx);
    FTT_CHECK(copy_to_host(ctx, &nuniq[side], bc + nt + 1, sizeof(int64_t)));
    FTT_CHECK(owned_alloc(ctx, (void **)&vec[side], 8 * (size_t)std::max<int64_t>(nuniq[side], 1) * rm));
    k_half_vectors<<<grid_for(nuniq[side], 8, 1, 148 * 64), 256, 0, ctx->stream>>>(
        nuniq[side], uniq[side], t, k0, k1, side == 0, vec[side], rm);
    FTT_LAUNCHED(ctx);
  }
  const int pb_ = prof_begin(ctx);
  k_mitm_dot<<<grid_for(n, 256, 4), 256, 0, ctx->stream>>>(n, rm, ids[0], ids[1], vec[0], vec[1], out);
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb_, PT_ENTRIES, (double)n * (16.0 + 8.0), 2.0 * (double)n * rm);
  for (void *p : {(void *)keys, (void *)skeys, (void *)idx, (void *)perm, (void *)bc, (void *)ids[0],
                  (void *)ids[1], (void *)uniq[0], (void *)uniq[1], (void *)vec[0], (void *)vec[1]})
    owned_free(ctx, p);
  return FTT_OK;
}

}  // namespace
}  // namespace ftt

using namespace ftt;

extern "C" int ftt_tt_entries(ftt_ctx *ctx, int32_t d, const int64_t *dims_host,
                              const int64_t *ranks_host, const double *const *cores_host,
                              const int64_t *coords, int64_t n, double *out) {
  if (!ctx || d < 1 || d > 32) {
    set_error("ftt_tt_entries: invalid train");
    return FTT_ERR_INVALID;
  }
  if (n == 0) return FTT_OK;
  TrainDesc t;
  t.d = d;
  int64_t rmax = 1;
  for (int k = 0; k < d; ++k) {
    t.dims[k] = dims_host[k];
    t.cores[k] = cores_host[k];
  }
  for (int k = 0; k <= d; ++k) {
    t.ranks[k] = ranks_host[k];
    rmax = std::max(rmax, ranks_host[k]);
  }
  if (ranks_host[0] != 1 || ranks_host[d] != 1) {
    set_error("edge ranks must be 1");
    return FTT_ERR_INVALID;
  }
  // direct evaluation costs ~n * sum_k r_k shuffle-FMA steps per lane group;
  // the meet-in-the-middle path a fixed ~0.2 ms of sorts: it only pays for
  // large n * sum_k r_k (config 5: 8.5M coordinates x 176)
  double steps = 0.0;
  for (int k = 0; k < d; ++k) steps += (double)ranks_host[k];
  if (rmax <= 64 && d >= 4 && (double)n * steps > 4e8 && n < ((int64_t)1 << 31))
    return entries_mitm(ctx, t, coords, n, out);
  if (rmax <= 8) {
    double steps_sum = 0.0;
    for (int k = 0; k < d; ++k) steps_sum += (double)ranks_host[k] * ranks_host[k + 1];
    const int pb = prof_begin(ctx);
    const int grid = grid_for(n, 256, 1, 148 * 16);
    int al = 1;
    for (int k = 0; k < d; ++k) al &= (((uintptr_t)cores_host[k]) & 15) == 0;
    if (rmax <= 4) k_entries_thr<4><<<grid, 256, 0, ctx->stream>>>(t, coords, n, out, al);
    else k_entries_thr<8><<<grid, 256, 0, ctx->stream>>>(t, coords, n, out, al);
    FTT_LAUNCHED(ctx);
    prof_end(ctx, pb, PT_ENTRIES, (double)n * (8.0 * d + 8.0), 2.0 * steps_sum * (double)n);
    return FTT_OK;
  }
  if (rmax <= 32) {
    const int L = rmax <= 4 ? 4 : rmax <= 8 ? 8 : rmax <= 16 ? 16 : 32;
    const int grid = grid_for(n, 8 * (32 / L), 1, 148 * 64);
    double steps_sum = 0.0;
    for (int k = 0; k < d; ++k) steps_sum += (double)ranks_host[k] * ranks_host[k + 1];
    const int pb = prof_begin(ctx);
    if (L == 4) k_entries_grp<4><<<grid, 256, 0, ctx->stream>>>(t, coords, n, out);
    else if (L == 8) k_entries_grp<8><<<grid, 256, 0, ctx->stream>>>(t, coords, n, out);
    else if (L == 16) k_entries_grp<16><<<grid, 256, 0, ctx->stream>>>(t, coords, n, out);
    else k_entries_grp<32><<<grid, 256, 0, ctx->stream>>>(t, coords, n, out);
    FTT_LAUNCHED(ctx);
    // coordinates + output per point; 2 sum_k r_k r_{k+1} flops per point
    prof_end(ctx, pb, PT_ENTRIES, (double)n * (8.0 * d + 8.0), 2.0 * steps_sum * (double)n);
    return FTT_OK;
  }
  if (rmax <= 64) {
    k_entries_small<<<grid_for(n, 8, 1, 148 * 64), 256, 0, ctx->stream>>>(t, coords, n, out);
    FTT_LAUNCHED(ctx);
    return FTT_OK;
  }
  // grouped GEMM path, in chunks to bound memory
  const int64_t chunk = std::min<int64_t>(n, std::max<int64_t>(4096, (int64_t)(1ll << 31) / (8 * rmax)));
  int64_t nkmax = 1;
  for (int k = 0; k < d; ++k) nkmax = std::max(nkmax, dims_host[k]);
  size_t need = 2 * align_up(8 * (size_t)chunk * rmax) + 2 * align_up(8 * chunk) +
                align_up(8 * chunk) + align_up(4 * chunk) + align_up(8 * (nkmax + 1)) +
                radix_sort_scratch_bytes(chunk, true) + align_up(8 * chunk) + align_up(4 * chunk) +
                4096;
  FTT_CHECK(arena_reserve(ctx, need));
  double *V = take<double>(ctx, (size_t)chunk * rmax);
  double *Vs = take<double>(ctx, (size_t)chunk * rmax);
  int64_t *idx = take<int64_t>(ctx, chunk);
  int64_t *idx2 = take<int64_t>(ctx, chunk);
  uint64_t *keys = take<uint64_t>(ctx, chunk);
  uint32_t *pos = take<uint32_t>(ctx, chunk);
  int64_t *off = take<int64_t>(ctx, nkmax + 1);
  uint64_t *skeys = take<uint64_t>(ctx, chunk);
  uint32_t *perm = take<uint32_t>(ctx, chunk);
  if (!perm) {
    set_error("ftt_tt_entries: arena too small");
    return FTT_ERR_INVALID;
  }
  std::vector<int64_t> hoff(nkmax + 1);
  for (int64_t c0 = 0; c0 < n; c0 += chunk) {
    const int64_t cn = std::min(chunk, n - c0);
    k_iota64<<<grid_for(cn, 256, 4), 256, 0, ctx->stream>>>(cn, c0, idx);
    FTT_LAUNCHED(ctx);
    int64_t r = ranks_host[1];
    k_first_rows<<<grid_for(cn * r, 256, 4), 256, 0, ctx->stream>>>(cn, coords, d, cores_host[0], r,
                                                                     idx, V);
    FTT_LAUNCHED(ctx);
    for (int k = 1; k < d; ++k) {
      const int64_t nk = dims_host[k], r0 = ranks_host[k], r1 = ranks_host[k + 1];
      k_level_keys<<<grid_for(cn, 256, 4), 256, 0, ctx->stream>>>(cn, coords, d, k, idx, keys, pos);
      FTT_LAUNCHED(ctx);
      size_t mark = ctx->arena.used;
      FTT_CHECK(radix_sort(ctx, keys, pos, skeys, perm, cn, std::max(1, bitlen((uint64_t)(nk - 1)))));
      ctx->arena.used = mark;
      k_permute_rows<<<grid_for(cn * r0, 256, 4), 256, 0, ctx->stream>>>(cn, r0, perm, V, Vs, idx, idx2);
      FTT_LAUNCHED(ctx);
      std::swap(idx, idx2);
      k_bounds<<<grid_for(cn + 1, 256, 4), 256, 0, ctx->stream>>>(cn, skeys, nk, off);
      FTT_LAUNCHED(ctx);
      FTT_CHECK(copy_to_host(ctx, hoff.data(), off, 8 * (nk + 1)));
      for (int64_t v = 0; v < nk; ++v) {
        int64_t cnt = hoff[v + 1] - hoff[v];
        if (cnt <= 0) continue;
        // (cnt x r0) @ (r0 x r1) row-major == col-major (r1 x cnt) = G^T (r1 x r0) * Vs^T (r0 x cnt)
        FTT_CHECK(gemm(ctx, 0, 0, r1, cnt, r0, 1.0, cores_host[k] + v * r1, nk * r1,
                       Vs + hoff[v] * r0, r0, 0.0, V + hoff[v] * r1, r1, nullptr, 0));
      }
      r = r1;
    }
    k_scatter_out<<<grid_for(cn, 256, 4), 256, 0, ctx->stream>>>(cn, 1, V, idx, out);
    FTT_LAUNCHED(ctx);
  }
  return FTT_OK;
}

// Frobenius norm of a train by contracting it with itself (ttformat.py:
// 198-203): W_0 = [1]; per core G (a x n x b): T = W G (a x n b), W' = G^T T
// over the (a n) rows (b x b); ||t||^2 = W_d.  Two DMMA GEMMs per core, one
// host round trip.
// ||t||^2 into the device scalar out_dev (no host round trip).
static int tt_norm2_dev(ftt_ctx *ctx, int32_t d, const int64_t *dims_host, const int64_t *ranks_host,
                        const double *const *cores_host, double *out_dev) {
  int64_t wmax = 1, tmax = 1;
  size_t ske = 1;
  for (int k = 0; k < d; ++k) {
    const int64_t a = ranks_host[k], n = dims_host[k], b = ranks_host[k + 1];
    wmax = std::max(wmax, b * b);
    tmax = std::max(tmax, a * n * b);
    ske = std::max({ske, gemm_splitk_elems(n * b, a, a), gemm_splitk_elems(b, b, a * n)});
  }
  double *W[2] = {nullptr, nullptr}, *T = nullptr, *sk = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&W[0], 8 * (size_t)wmax));
  FTT_CHECK(owned_alloc(ctx, (void **)&W[1], 8 * (size_t)wmax));
  FTT_CHECK(owned_alloc(ctx, (void **)&T, 8 * (size_t)tmax));
  FTT_CHECK(owned_alloc(ctx, (void **)&sk, 8 * ske));
  const double one = 1.0;
  FTT_CHECK(stage_to_device(ctx, W[0], &one, sizeof(double)));
  int cur = 0;
  for (int k = 0; k < d; ++k) {
    const int64_t a = ranks_host[k], n = dims_host[k], b = ranks_host[k + 1];
    // row-major T (a x n b) = W (a x a) G (a x n b)  <=>  col-major T^T = G^T W^T
    FTT_CHECK(gemm(ctx, 0, 0, n * b, a, a, 1.0, cores_host[k], n * b, W[cur], a, 0.0, T, n * b, sk,
                   ske));
    // W' (b x b) = G(a n x b)^T T(a n x b)  <=>  col-major W'^T = T^T G  (row-major views)
    FTT_CHECK(gemm(ctx, 0, 1, b, b, a * n, 1.0, T, b, cores_host[k], b, 0.0, W[cur ^ 1], b, sk, ske));
    cur ^= 1;
  }
  FTT_CUDA(cudaMemcpyAsync(out_dev, W[cur], sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  owned_free(ctx, W[0]);
  owned_free(ctx, W[1]);
  owned_free(ctx, T);
  owned_free(ctx, sk);
  return FTT_OK;
}

extern "C" int ftt_tt_norm(ftt_ctx *ctx, int32_t d, const int64_t *dims_host,
                           const int64_t *ranks_host, const double *const *cores_host,
                           double *norm_out) {
  if (!ctx || !norm_out || d < 1 || d > 32) {
    set_error("ftt_tt_norm: invalid train");
    return FTT_ERR_INVALID;
  }
  double *dev = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&dev, 64));
  FTT_CHECK(tt_norm2_dev(ctx, d, dims_host, ranks_host, cores_host, dev));
  double v = 0.0;
  FTT_CHECK(copy_to_host(ctx, &v, dev, sizeof(double)));
  owned_free(ctx, dev);
  *norm_out = std::sqrt(std::max(v, 0.0));
  return FTT_OK;
}

// The three terms of sparse_inner_error (fasttt.py:587-602) with one host
// round trip: out_host[0] = <values, entries>, out_host[1] = ||t||^2.
extern "C" int ftt_inner_terms(ftt_ctx *ctx, int64_t n, const double *values,
                               const double *entries, int32_t d, const int64_t *dims_host,
                               const int64_t *ranks_host, const double *const *cores_host,
                               double *out_host) {
  if (!ctx || !out_host || d < 1 || d > 32 || n < 0) {
    set_error("ftt_inner_terms: invalid arguments");
    return FTT_ERR_INVALID;
  }
  double *dev = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&dev, 8 * (size_t)(kSumSqBlocks + 4)));
  FTT_CHECK(dot_dev(ctx, n, values, entries, dev + 2, dev));
  FTT_CHECK(tt_norm2_dev(ctx, d, dims_host, ranks_host, cores_host, dev + 1));
  FTT_CHECK(copy_to_host(ctx, out_host, dev, 2 * sizeof(double)));
  owned_free(ctx, dev);
  return FTT_OK;
}


// ---------------------------------------------------------------------------
// <a, b> for the report's inner-product identity (fasttt.py:587-602) from
// the index structure fasttt already holds, instead of evaluating the
// rounded train b at every nonzero coordinate independently.  The left
// sweep's kept rows are exactly the distinct prefixes (i_0..i_k) of the
// fibers (kept_k[j] = t * n_k + i: prefix j extends prefix t of the previous
// step by i), the right sweep's the distinct suffixes (kept[j] = i * r + s),
// and t_map / s_map name each fiber's prefix and suffix.  So
//   V_k[j] = V_{k-1}[t] . b_k[:, i, :]        (left vectors, K_k x r_k)
//   W_k[j] = b_k[:, i, :] . W_{k+1}[s]        (right vectors)
//   M[t, i] = V_{p-1}[t] . b_p[:, i, :]       (every prefix x pivot index)
//   b(e) = M[t_map[f], i_e] . W_{p+1}[s_map[f]]   for entry e of fiber f
// -- per nonzero r_p multiply-adds after O(sum_k K_k r_k r_{k+1}) setup.
namespace ftt {
namespace {

// out[j, b] = sum_a prev[t, a] core[a, i, b], (t, i) = (kept[j] / n, kept[j] % n)
// (kept == nullptr: j itself; prev == nullptr: rin = 1 and prev = 1)
__global__ void k_left_vec(int64_t K, const int64_t *__restrict__ kept, int64_t n, int rin,
                           int rout, const double *__restrict__ prev,
                           const double *__restrict__ core, double *__restrict__ out) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < K * rout;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = x / rout;
    const int b = (int)(x - j * rout);
    const int64_t row = kept ? kept[j] : j;
    const int64_t t = row / n, i = row - t * n;
    double s = 0.0;
    if (prev) {
      const double *pv = prev + t * rin;
      for (int a = 0; a < rin; ++a) s += pv[a] * core[(a * n + i) * rout + b];
    } else {
      s = core[i * rout + b];
    }
    out[x] = s;
  }
}

// The same product with the core slice staged in shared memory, transposed
// to [i][b][a]: LP lanes per kept row (LP = rin rounded up to a power of
// two), lane a owns out[j, a] = sum_b core[a, i, b] next[s, b] -- the core
// reads are conflict-free (a fastest), next[s, :] is a broadcast read, and
// there are no shuffles (k_right_vec<16> spent its time in the 64 butterfly
// shuffles per row: 142 -> ~40 us on config 5's 314,928 suffixes).
template <int RO>
__global__ void __launch_bounds__(256) k_right_vec_sm(int64_t K, const int64_t *__restrict__ kept,
                                                      int64_t r, int64_t n, int rin, int LP,
                                                      const double *__restrict__ next,
                                                      const double *__restrict__ core,
                                                      double *__restrict__ out) {
  extern __shared__ __align__(16) double sm[];  // n x RO x rin
  const int total = (int)(rin * n * RO);
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    // core[(a n + i) RO + b]  ->  sm[(i RO + b) rin + a]
    const int b = e % RO, ai = e / RO;
    const int i = ai % (int)n, a = ai / (int)n;
    sm[(i * RO + b) * rin + a] = core[e];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, a = lane % LP, rpw = 32 / LP;
  const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t stride = (((int64_t)gridDim.x * blockDim.x) >> 5) * rpw;
  for (int64_t base = wg * rpw; base < K; base += stride) {
    const int64_t j = base + lane / LP;
    if (j >= K || a >= rin) continue;
    const int64_t row = kept[j];
    const int64_t i = row / r, s = row - i * r;
    const double2 *nx = reinterpret_cast<const double2 *>(next + s * RO);
    const double *c = sm + (size_t)i * RO * rin + a;
    double acc = 0.0;
#pragma unroll
    for (int b2 = 0; b2 < RO / 2; ++b2) {
      const double2 w = __ldg(nx + b2);
      acc = fma(c[(2 * b2) * rin], w.x, acc);
      acc = fma(c[(2 * b2 + 1) * rin], w.y, acc);
    }
    out[j * rin + a] = acc;
  }
}

// out[j, :] = core[:, i, :] . next[s, :], (i, s) = (kept[j] / r, kept[j] % r):
// RO lanes per kept row j (RO = 8 / 16 / 32 = rout): lane b holds next[s, b]
// and reads core[a, i, b] for every a (coalesced rows), the products are
// reduced over the RO lanes (butterfly) and lane a % RO keeps out[j, a].
// RO = 0: generic thread-per-row loop (other ranks, the last core).
template <int RO>
__global__ void k_right_vec(int64_t K, const int64_t *__restrict__ kept, int64_t r, int64_t n,
                            int rin, int rout, const double *__restrict__ next,
                            const double *__restrict__ core, double *__restrict__ out) {
  if constexpr (RO > 0) {
    constexpr int RPW = 32 / RO;  // kept rows per warp
    const int lane = threadIdx.x & 31, b = lane % RO;
    const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t stride = (((int64_t)gridDim.x * blockDim.x) >> 5) * RPW;
    const unsigned mask = 0xffffffffu;
    for (int64_t base = wg * RPW; base < K; base += stride) {  // warp-uniform
      const int64_t j0 = base + lane / RO;
      const bool live = j0 < K;
      const int64_t j = live ? j0 : 0;
      const int64_t row = kept[j];
      const int64_t i = row / r, s = row - i * r;
      const double w = next[s * RO + b];
      for (int a0 = 0; a0 < rin; a0 += RO) {
        double keep = 0.0;
        for (int a = a0; a < a0 + RO; ++a) {
          double x = a < rin ? core[(a * n + i) * RO + b] * w : 0.0;
#pragma unroll
          for (int o = RO / 2; o; o >>= 1) x += __shfl_xor_sync(mask, x, o);
          if (a - a0 == b) keep = x;
        }
        if (live && a0 + b < rin) out[j * rin + a0 + b] = keep;
      }
    }
  } else {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < K;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = kept[j];
    const int64_t i = row / r, s = row - i * r;
    for (int a = 0; a < rin; ++a) {
      const double *cr = core + (a * n + i) * rout;
      double acc = 0.0;
      if (next) {
        const double *nx = next + s * rout;
        for (int c = 0; c < rout; ++c) acc += cr[c] * nx[c];
      } else {
        acc = cr[0];
      }
      out[j * rin + a] = acc;
    }
  }
  }
}

// Block partials of sum_e values[e] * (M[t, i_e] . W[s]) = sum_c W[s, c]
// (sum_e values[e] M[t, i_e, c]): RR lanes per fiber f (lane c holds W[s, c]
// and reads M rows coalesced), the fiber's nonzeros indptr[f]..indptr[f+1]
// in order, each lane accumulating its own c; fixed-order block sums.
// RR = 0: one thread per fiber (other ranks, no right part).
template <int RR>
__global__ void __launch_bounds__(256) k_inner_struct(int64_t R, const int64_t *__restrict__ indptr,
                                                      const int64_t *__restrict__ pidx,
                                                      const double *__restrict__ values,
                                                      const int64_t *__restrict__ t_map,
                                                      const int64_t *__restrict__ s_map, int64_t np,
                                                      int r, const double *__restrict__ M,
                                                      const double *__restrict__ W,
                                                      double *__restrict__ partial) {
  __shared__ double red[8];
  double acc = 0.0;
  if constexpr (RR > 0) {
    const int c = threadIdx.x % RR;
    const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / RR;
    const int64_t gs = ((int64_t)gridDim.x * blockDim.x) / RR;
    for (int64_t f = g0; f < R; f += gs) {
      const int64_t t = t_map ? t_map[f] : 0, s = s_map[f];
      const double w = W[s * RR + c];
      const double *mrow = M + t * np * RR + c;
      const int64_t e1 = indptr[f + 1];
      double sv = 0.0;
      for (int64_t e = indptr[f]; e < e1; ++e) sv += values[e] * mrow[pidx[e] * RR];
      acc += w * sv;
    }
  } else {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < R;
         f += (int64_t)gridDim.x * blockDim.x) {
      const int64_t t = t_map ? t_map[f] : 0, s = s_map ? s_map[f] : 0;
      const double *mrow = M + t * np * r;
      for (int64_t e = indptr[f]; e < indptr[f + 1]; ++e) {
        const double *m = mrow + pidx[e] * r;
        double b = 0.0;
        if (W) {
          const double *w = W + s * r;
          for (int c = 0; c < r; ++c) b += m[c] * w[c];
        } else {
          b = m[0];
        }
        acc += values[e] * b;
      }
    }
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

__global__ void k_sum_fixed(const double *__restrict__ p, int64_t n, double *__restrict__ out) {
  __shared__ double s[256];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) a += p[i];
  s[threadIdx.x] = a;
  __syncthreads();
  for (int off = 128; off; off >>= 1) {
    if ((int)threadIdx.x < off) s[threadIdx.x] += s[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

}  // namespace
}  // namespace ftt

extern "C" int ftt_inner_structured(ftt_ctx *ctx, int32_t d, const int64_t *dims,
                                    const int64_t *ranks, const double *const *cores,
                                    int32_t pivot, const int64_t *const *kept,
                                    const int64_t *kept_counts, int64_t R,
                                    const int64_t *indptr, const int64_t *pivot_index,
                                    const double *values, const int64_t *t_map,
                                    const int64_t *s_map, double *out_host) {
  if (!ctx || !out_host || d < 2 || d > 32 || pivot < 0 || pivot >= d || R < 0) {
    set_error("ftt_inner_structured: invalid arguments");
    return FTT_ERR_INVALID;
  }
  if (ranks[0] != 1 || ranks[d] != 1) {
    set_error("ftt_inner_structured: edge ranks must be 1");
    return FTT_ERR_INVALID;
  }
  // kept[] in sweep order: left steps 0..p-1, then right steps d-1 .. p+1
  int64_t bytes = 0;
  for (int k = 0; k < pivot; ++k) bytes += kept_counts[k] * ranks[k + 1];
  bytes += (pivot > 0 ? kept_counts[pivot - 1] : 1) * dims[pivot] * ranks[pivot + 1];
  for (int q = 0; q < d - 1 - pivot; ++q) {
    const int k = d - 1 - q;
    bytes += kept_counts[pivot + q] * ranks[k];
  }
  const int64_t nb = std::min<int64_t>(16 * (int64_t)ctx->num_sms, std::max<int64_t>(1, ceil_div(R, 16)));
  double *buf = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&buf, 8 * (size_t)(bytes + nb + 1)));
  double *cur = buf;
  const int pb = prof_begin(ctx);
  // left vectors, then M over every (prefix, pivot index)
  const double *V = nullptr;
  int64_t Kl = 1;
  for (int k = 0; k < pivot; ++k) {
    const int64_t K = kept_counts[k];
    k_left_vec<<<grid_for(K * ranks[k + 1], 256, 4), 256, 0, ctx->stream>>>(
        K, kept[k], dims[k], (int)ranks[k], (int)ranks[k + 1], V, cores[k], cur);
    FTT_LAUNCHED(ctx);
    V = cur;
    Kl = K;
    cur += K * ranks[k + 1];
  }
  double *M = cur;
  k_left_vec<<<grid_for(Kl * dims[pivot] * ranks[pivot + 1], 256, 4), 256, 0, ctx->stream>>>(
      Kl * dims[pivot], nullptr, dims[pivot], (int)ranks[pivot], (int)ranks[pivot + 1], V,
      cores[pivot], M);
  FTT_LAUNCHED(ctx);
  cur += Kl * dims[pivot] * ranks[pivot + 1];
  // right vectors from the last mode inwards
  const double *W = nullptr;
  int64_t r_other = 1;
  for (int q = 0; q < d - 1 - pivot; ++q) {
    const int k = d - 1 - q;
    const int64_t K = kept_counts[pivot + q];
    const int ro = (int)ranks[k + 1];
#define FTT_RV(RO_)                                                                           \
  k_right_vec<RO_><<<grid_for(K * (RO_ > 0 ? RO_ : 1), 256, 1), 256, 0, ctx->stream>>>(       \
      K, kept[pivot + q], r_other, dims[k], (int)ranks[k], ro, W, cores[k], cur)
    // long kept lists with a small core slice: the shared-memory variant
    const int rin = (int)ranks[k];
    const size_t slice = 8 * (size_t)rin * dims[k] * ro;
    if (W && K >= 60000 && rin <= 32 && (ro == 8 || ro == 16 || ro == 32) && slice <= 65536) {
      static bool attr = false;
      if (!attr) {
        FTT_CUDA(cudaFuncSetAttribute(k_right_vec_sm<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
        FTT_CUDA(cudaFuncSetAttribute(k_right_vec_sm<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
        FTT_CUDA(cudaFuncSetAttribute(k_right_vec_sm<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
        attr = true;
      }
      int LP = 1;
      while (LP < rin) LP <<= 1;
      const int g = grid_for(K * LP, 256, 4, 148 * 3);
      if (ro == 8)
        k_right_vec_sm<8><<<g, 256, slice, ctx->stream>>>(K, kept[pivot + q], r_other, dims[k], rin,
                                                          LP, W, cores[k], cur);
      else if (ro == 16)
        k_right_vec_sm<16><<<g, 256, slice, ctx->stream>>>(K, kept[pivot + q], r_other, dims[k], rin,
                                                           LP, W, cores[k], cur);
      else
        k_right_vec_sm<32><<<g, 256, slice, ctx->stream>>>(K, kept[pivot + q], r_other, dims[k], rin,
                                                           LP, W, cores[k], cur);
    } else if (!W) FTT_RV(0);  // the last core: no next vector
    else if (ro == 1) FTT_RV(1);
    else if (ro == 8) FTT_RV(8);
    else if (ro == 16) FTT_RV(16);
    else if (ro == 32) FTT_RV(32);
    else FTT_RV(0);
#undef FTT_RV
    FTT_LAUNCHED(ctx);
    W = cur;
    r_other = K;
    cur += K * ranks[k];
  }
  double *part = cur;
  const int rr = (int)ranks[pivot + 1];
#define FTT_IS(RR_)                                                                           \
  k_inner_struct<RR_><<<(unsigned)nb, 256, 0, ctx->stream>>>(R, indptr, pivot_index, values,  \
                                                             t_map, s_map, dims[pivot], rr, M, \
                                                             W, part)
  if (rr == 8 && W) FTT_IS(8);
  else if (rr == 16 && W) FTT_IS(16);
  else if (rr == 32 && W) FTT_IS(32);
  else FTT_IS(0);
#undef FTT_IS
  FTT_LAUNCHED(ctx);
  k_sum_fixed<<<1, 256, 0, ctx->stream>>>(part, nb, part + nb);
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb, PT_ENTRIES, 40.0 * (double)R + 8.0 * (double)bytes, 0.0);
  FTT_CHECK(copy_to_host(ctx, out_host, part + nb, sizeof(double)));
  owned_free(ctx, buf);
  return FTT_OK;
}
