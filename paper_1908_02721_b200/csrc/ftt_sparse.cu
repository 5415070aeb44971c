// Sparse operand for the first truncation step of the rounding sweep.
//
// The pivot core of parallel_vector_round (fasttt.py:256-259) holds exactly
// the nonzeros of the input: entry (t_map[f], i_p, s_map[f]) = value.  Its
// first SVD operand M = core.reshape(r_prev * n_p, r_next) is therefore a
// sparse matrix (config 5: 8.5M entries in 4160 x 314928, 0.65 % dense,
// 10.5 GB when densified).  The certified low-rank path only needs three
// products with the operand -- the sketch Y = A Omega, B = Q^T A and the
// residual energy ||A - Q B||_F^2 -- so it runs on the entries:
//
//   entries -> (row, col) of A_tall (= M, or M^T when M is wide); two stable
//   radix sorts give CSR (by row) and CSC (by column, rows ascending) orders
//   Y   : one warp per row, lanes over the sketch columns (Omega row-major)
//   B   : columns cut into segments of SEG entries (the pivot core's columns
//         are heavily skewed), one warp per segment with lanes over entries
//         (Q row-major), then a fixed-order sum of each column's segments
//   rest2 = S1 + S2, both sums of squares evaluated directly:
//         S1 = sum over the positions (r, c) NOT holding an entry of
//              (Q B)_rc^2: every element of Q B is formed (kr FMAs; B column
//              in registers, Q rows broadcast from shared memory) and an
//              occupancy bitmap (row-major, one 32-column word per warp and
//              row) masks the entries out;
//         S2 = sum over the entries of (A_rc - (Q B)_rc)^2.
//         The residual is never formed as a difference of two large sums
//         (that would cancel far above the certificate's 1e-6 delta^2
//         resolution).
// Every reduction has a fixed order: results are bit-reproducible.
#include "ftt_dense.cuh"

namespace ftt {
namespace {

__global__ void k_sp_entries(int64_t nnz, const int64_t *__restrict__ fiber_of,
                             const int64_t *__restrict__ pidx, const int64_t *__restrict__ tmap,
                             const int64_t *__restrict__ smap, int64_t np, int transposed,
                             int64_t mA, int32_t *__restrict__ ra, int32_t *__restrict__ ca,
                             uint64_t *__restrict__ key_r, uint64_t *__restrict__ key_c,
                             uint32_t *__restrict__ ident) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = fiber_of[e];
    const int64_t row = (tmap ? tmap[f] : 0) * np + pidx[e];
    const int64_t col = smap ? smap[f] : 0;
    const int64_t r = transposed ? col : row, c = transposed ? row : col;
    ra[e] = (int32_t)r;
    ca[e] = (int32_t)c;
    key_r[e] = (uint64_t)r;
    key_c[e] = (uint64_t)c * (uint64_t)mA + (uint64_t)r;
    ident[e] = (uint32_t)e;
  }
}

// ptr[i] = first p with keys[p] >= i * scale, i in [0, count] (keys sorted).
__global__ void k_lower_bounds(const uint64_t *__restrict__ keys, int64_t n, int64_t count,
                               uint64_t scale, int64_t *__restrict__ ptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t target = (uint64_t)i * scale;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    ptr[i] = lo;
  }
}

__global__ void k_sp_gather(int64_t n, const uint32_t *__restrict__ perm,
                            const int32_t *__restrict__ idx_in, const double *__restrict__ v_in,
                            int32_t *__restrict__ idx_out, double *__restrict__ v_out) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t e = perm[p];
    if (idx_out) idx_out[p] = idx_in[e];
    v_out[p] = v_in[e];
  }
}

// The range finder's test matrix (same values as k_omega in ftt_svd.cu,
// element (c, j) = splitmix64(c + j nA)) stored row-major nA x k.
__global__ void k_omega_rows(int64_t nA, int k, double *__restrict__ Or) {
  const int64_t total = nA * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / k, j = t - c * k;
    uint64_t z = (uint64_t)(c + j * nA) + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    Or[t] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
}

// Y = A_tall Omega (mA x k col-major): one warp per row, lanes j and j + 32.
__global__ void __launch_bounds__(256) k_spmm_rows(int64_t mA, int k, const int64_t *__restrict__ rptr,
                                                   const int32_t *__restrict__ cidx,
                                                   const double *__restrict__ v,
                                                   const double *__restrict__ Or,
                                                   double *__restrict__ Y) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < mA; r += warps) {
    const int64_t e0 = rptr[r], e1 = rptr[r + 1];
    double a0 = 0.0, a1 = 0.0;
    int64_t e = e0;
    for (; e + 4 <= e1; e += 4) {  // four entries' loads in flight together
      int32_t c[4];
      double w[4], o0[4], o1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] = cidx[e + u];
        w[u] = v[e + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double *row = Or + (int64_t)c[u] * k;
        o0[u] = lane < k ? row[lane] : 0.0;
        o1[u] = lane + 32 < k ? row[lane + 32] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0 += w[u] * o0[u];
        a1 += w[u] * o1[u];
      }
    }
    for (; e < e1; ++e) {
      const double *row = Or + (int64_t)cidx[e] * k;
      const double w = v[e];
      if (lane < k) a0 += w * row[lane];
      if (lane + 32 < k) a1 += w * row[lane + 32];
    }
    if (lane < k) Y[r + (int64_t)lane * mA] = a0;
    if (lane + 32 < k) Y[r + (int64_t)(lane + 32) * mA] = a1;
  }
}

// Column segments of the CSC order: seg_cnt[c] = ceil(len_c / SEG).
constexpr int SEG = 1024;
__global__ void k_seg_counts(int64_t nA, const int64_t *__restrict__ cptr, int64_t *__restrict__ cnt) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nA;
       c += (int64_t)gridDim.x * blockDim.x)
    cnt[c] = (cptr[c + 1] - cptr[c] + SEG - 1) / SEG;
}

// Partial B columns: one warp per segment (global index g; its column is
// the last c with seg_base[c] <= g), lanes over the segment's entries,
// fixed-order butterfly; partial[g * kr + j].
template <int KR>
__global__ void __launch_bounds__(256) k_spmm_seg(int64_t nA, int kr, int ldq, int64_t max_segs,
                                                  const int64_t *__restrict__ cptr,
                                                  const int64_t *__restrict__ seg_base,
                                                  const int32_t *__restrict__ ridx,
                                                  const double *__restrict__ v,
                                                  const double *__restrict__ Qr,
                                                  double *__restrict__ partial) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t total = seg_base[nA];
  for (int64_t g = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); g < max_segs && g < total;
       g += warps) {
    int64_t lo = 0, hi = nA;  // last c with seg_base[c] <= g (and a non-empty column)
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (seg_base[mid] <= g) lo = mid;
      else hi = mid;
    }
    const int64_t c = lo;
    const int64_t e0 = cptr[c] + (g - seg_base[c]) * SEG;
    const int64_t e1 = min(cptr[c + 1], e0 + SEG);
    double acc[KR];
#pragma unroll
    for (int j = 0; j < KR; ++j) acc[j] = 0.0;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const double w = v[e];
      // Q row as 16-byte pairs (ldq even; entries kr..ldq-1 of a row are zero)
      const double2 *q = reinterpret_cast<const double2 *>(Qr + (int64_t)ridx[e] * ldq);
#pragma unroll
      for (int j = 0; j < KR; j += 2)
        if (j < kr) {
          const double2 t = __ldg(q + j / 2);
          acc[j] += w * t.x;
          acc[j + 1] += w * t.y;
        }
    }
#pragma unroll
    for (int j = 0; j < KR; ++j) {
      double s = acc[j];
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      acc[j] = s;
    }
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < KR; ++j)
        if (j < kr) partial[g * kr + j] = acc[j];
    }
  }
}

// B[j, c] = sum of the column's segment partials in segment order.
__global__ void k_seg_reduce(int64_t nA, int kr, const int64_t *__restrict__ seg_base,
                             const double *__restrict__ partial, double *__restrict__ B) {
  const int64_t total = nA * kr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / kr, j = t - c * kr;
    double s = 0.0;
    for (int64_t g = seg_base[c]; g < seg_base[c + 1]; ++g) s += partial[g * kr + j];
    B[j + c * kr] = s;
  }
}

// Occupancy bitmap of A_tall, row-major with the columns padded to 32:
// bit (r, c) = word r * wpr + c / 32, bit c % 32.
__global__ void k_sp_bitmap(int64_t nnz, const int32_t *__restrict__ ridx,
                            const int32_t *__restrict__ cidx, int64_t wpr, unsigned *__restrict__ bm) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = ridx[e], c = cidx[e];
    atomicOr(bm + r * wpr + (c >> 5), 1u << (c & 31));
  }
}

// S1 partials: CTA = (64-column block, row chunk).  The block's B columns
// sit in shared memory; every lane holds ROWS rows of Q (row-major copy) in
// registers and walks the 64 columns: per column one broadcast read of the
// B column (conflict-free), kr FMAs per row, and the occupancy bit of
// (row, column) from the row's two bitmap words masks out positions holding
// an entry.  One barrier per CTA; no long-latency load in the column loop.
constexpr int RCB = 64;  // columns per CTA
template <int KR, int ROWS>
__global__ void __launch_bounds__(256) k_sp_resid_off(int64_t mA, int64_t nA, int kr, int ldq,
                                                      const double *__restrict__ Qr,
                                                      const double *__restrict__ B,
                                                      const unsigned *__restrict__ bm, int64_t wpr,
                                                      int64_t chunk, double *__restrict__ partial) {
  __shared__ __align__(16) double Bs[RCB][KR];
  __shared__ double red[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * RCB;
  const int ncol = (int)min((int64_t)RCB, nA - c0);
  for (int e = threadIdx.x; e < RCB * KR; e += blockDim.x) {
    const int cc = e / KR, j = e - cc * KR;
    Bs[cc][j] = (cc < ncol && j < kr) ? B[j + (c0 + cc) * (int64_t)kr] : 0.0;
  }
  __syncthreads();
  const int64_t rbeg = (int64_t)blockIdx.y * chunk, rend = min(mA, rbeg + chunk);
  const int64_t wg = c0 >> 5;  // first bitmap word of the block
  double acc = 0.0;
  for (int64_t base = rbeg + (int64_t)w * 32 * ROWS; base < rend; base += 8 * 32 * ROWS) {
    double qv[ROWS][KR];
    unsigned wd[ROWS][2];
    bool live[ROWS];
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      const int64_t r = base + lane + 32 * i;
      live[i] = r < rend;
      const double *q = Qr + (live[i] ? r : 0) * ldq;  // ldq even: 16-byte rows
#pragma unroll
      for (int j = 0; j < KR; j += 2) {
        double2 t = make_double2(0.0, 0.0);
        if (live[i] && j < kr) t = __ldg(reinterpret_cast<const double2 *>(q + j));
        qv[i][j] = t.x;
        qv[i][j + 1] = t.y;
      }
      const unsigned *wp = bm + (live[i] ? r : 0) * wpr + wg;
      wd[i][0] = live[i] ? __ldg(wp) : ~0u;
      wd[i][1] = (live[i] && wg + 1 < wpr) ? __ldg(wp + 1) : ~0u;
    }
#pragma unroll 2
    for (int cc = 0; cc < ncol; ++cc) {
      double bv[KR];
#pragma unroll
      for (int j = 0; j < KR; j += 2) {
        const double2 t = *reinterpret_cast<const double2 *>(&Bs[cc][j]);
        bv[j] = t.x;
        bv[j + 1] = t.y;
      }
#pragma unroll
      for (int i = 0; i < ROWS; ++i) {
        double qb = 0.0;
#pragma unroll
        for (int j = 0; j < KR; ++j) qb += qv[i][j] * bv[j];
        const unsigned bit = (wd[i][cc >> 5] >> (cc & 31)) & 1u;
        if (!bit) acc += qb * qb;
      }
    }
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if (lane == 0) red[w] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += red[i];
    partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

// S2 partials: (A_rc - (Q B)_rc)^2 over the entries (CSC arrays), a fixed
// entry range per block.
template <int KR>
__global__ void __launch_bounds__(256) k_sp_resid_on(int64_t nnz, int kr, int ldq,
                                                     const int32_t *__restrict__ ridx,
                                                     const int32_t *__restrict__ cidx,
                                                     const double *__restrict__ v,
                                                     const double *__restrict__ Qr,
                                                     const double *__restrict__ B, int64_t per,
                                                     double *__restrict__ partial) {
  __shared__ double red[8];
  const int64_t e0 = (int64_t)blockIdx.x * per, e1 = min(nnz, e0 + per);
  double acc = 0.0;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const double2 *q = reinterpret_cast<const double2 *>(Qr + (int64_t)ridx[e] * ldq);
    const double *bc = B + (int64_t)cidx[e] * kr;
    double qb = 0.0;
#pragma unroll
    for (int j = 0; j < KR; j += 2)
      if (j < kr) {
        const double2 t = __ldg(q + j / 2);
        qb += t.x * bc[j];
        if (j + 1 < kr) qb += t.y * bc[j + 1];
      }
    const double d = v[e] - qb;
    acc += d * d;
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < 8; ++i) s += red[i];
    partial[blockIdx.x] = s;
  }
}

__global__ void k_sp_sum(const double *__restrict__ p, int64_t n, double *__restrict__ out) {
  __shared__ double s[1024];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a += p[i];
  s[threadIdx.x] = a;
  __syncthreads();
  for (int off = blockDim.x / 2; off; off >>= 1) {
    if ((int)threadIdx.x < off) s[threadIdx.x] += s[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

__global__ void k_gather_i32(int64_t n, const uint32_t *__restrict__ perm, const int32_t *__restrict__ in,
                             int32_t *__restrict__ out) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    out[p] = in[perm[p]];
}

// Exclusive scan of n int64 counts into out[0..n] (out[n] = total): block
// scans of 1024, a scan of the block totals, then the offsets.
__global__ void __launch_bounds__(1024) k_scan_blocks(const int64_t *__restrict__ in, int64_t n,
                                                      int64_t *__restrict__ out,
                                                      int64_t *__restrict__ btot) {
  __shared__ int64_t sh[1024];
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const int64_t x = i < n ? in[i] : 0;
  sh[threadIdx.x] = x;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int64_t y = threadIdx.x >= off ? sh[threadIdx.x - off] : 0;
    __syncthreads();
    sh[threadIdx.x] += y;
    __syncthreads();
  }
  if (i < n) out[i] = sh[threadIdx.x] - x;
  if (threadIdx.x == 1023) btot[blockIdx.x] = sh[1023];
}

__global__ void k_scan_fix(int64_t n, int64_t nb, int64_t *__restrict__ out,
                           const int64_t *__restrict__ btot) {
  // one block: serial prefix of the (few) block totals in shared memory
  extern __shared__ int64_t off[];
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int64_t b = 0; b < nb; ++b) {
      off[b] = run;
      run += btot[b];
    }
    out[n] = run;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[i] += off[i / 1024];
}

int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return b;
}

}  // namespace

int sparse_operand_build(ftt_ctx *ctx, SparseOperand *op, int64_t nnz, const int64_t *fiber_of,
                         const int64_t *pidx, const double *vals, const int64_t *tmap,
                         const int64_t *smap, int64_t np, int64_t m, int64_t n) {
  op->nnz = nnz;
  op->transposed = m < n;
  op->mA = std::max(m, n);
  op->nA = std::min(m, n);
  const int64_t mA = op->mA, nA = op->nA;
  int32_t *ra = nullptr, *ca = nullptr;
  uint64_t *key_r = nullptr, *key_c = nullptr, *sorted = nullptr;
  uint32_t *ident = nullptr, *perm = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&ra, 4 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&ca, 4 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&key_r, 8 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&key_c, 8 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&ident, 4 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&perm, 4 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->rptr, 8 * (size_t)(mA + 1)));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->cptr, 8 * (size_t)(nA + 1)));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->cidx_r, 4 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->v_r, 8 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->keyc, 8 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->v_c, 8 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->ridx_c, 4 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->cidx_c, 4 * (size_t)nnz));
  const int pb = prof_begin(ctx);
  k_sp_entries<<<grid_for(nnz, 256, 4), 256, 0, ctx->stream>>>(
      nnz, fiber_of, pidx, tmap, smap, np, op->transposed ? 1 : 0, mA, ra, ca, key_r, key_c, ident);
  FTT_LAUNCHED(ctx);
  // CSR: stable sort by row (entries of a row keep the fiber order)
  FTT_CHECK(arena_reserve(ctx, radix_sort_scratch_bytes(nnz, true) + 4096));
  FTT_CHECK(owned_alloc(ctx, (void **)&sorted, 8 * (size_t)nnz));
  FTT_CHECK(radix_sort(ctx, key_r, ident, sorted, perm, nnz, bits_for((uint64_t)(mA - 1))));
  k_lower_bounds<<<grid_for(mA + 1, 256, 4), 256, 0, ctx->stream>>>(sorted, nnz, mA, 1, op->rptr);
  FTT_LAUNCHED(ctx);
  k_sp_gather<<<grid_for(nnz, 256, 4), 256, 0, ctx->stream>>>(nnz, perm, ca, vals, op->cidx_r, op->v_r);
  FTT_LAUNCHED(ctx);
  // CSC: sort by (column, row)
  FTT_CHECK(arena_reserve(ctx, radix_sort_scratch_bytes(nnz, true) + 4096));
  FTT_CHECK(radix_sort(ctx, key_c, ident, op->keyc, perm, nnz,
                       bits_for((uint64_t)nA * (uint64_t)mA - 1)));
  k_lower_bounds<<<grid_for(nA + 1, 256, 4), 256, 0, ctx->stream>>>(op->keyc, nnz, nA,
                                                                     (uint64_t)mA, op->cptr);
  FTT_LAUNCHED(ctx);
  k_sp_gather<<<grid_for(nnz, 256, 4), 256, 0, ctx->stream>>>(nnz, perm, ra, vals, op->ridx_c, op->v_c);
  FTT_LAUNCHED(ctx);
  k_gather_i32<<<grid_for(nnz, 256, 4), 256, 0, ctx->stream>>>(nnz, perm, ca, op->cidx_c);
  FTT_LAUNCHED(ctx);
  // column segments (B = Q^T A is computed per segment: the columns are skewed)
  {
    int64_t *cnt = nullptr, *btot = nullptr;
    const int64_t nb = ceil_div(nA, 1024);
    if (nb > 6000) {
      set_error("sparse operand: too many columns");
      return FTT_ERR_INVALID;
    }
    FTT_CHECK(owned_alloc(ctx, (void **)&cnt, 8 * (size_t)nA));
    FTT_CHECK(owned_alloc(ctx, (void **)&btot, 8 * (size_t)nb));
    FTT_CHECK(owned_alloc(ctx, (void **)&op->seg_base, 8 * (size_t)(nA + 1)));
    k_seg_counts<<<grid_for(nA, 256, 4), 256, 0, ctx->stream>>>(nA, op->cptr, cnt);
    FTT_LAUNCHED(ctx);
    k_scan_blocks<<<(unsigned)nb, 1024, 0, ctx->stream>>>(cnt, nA, op->seg_base, btot);
    FTT_LAUNCHED(ctx);
    k_scan_fix<<<1, 1024, 8 * (size_t)nb, ctx->stream>>>(nA, nb, op->seg_base, btot);
    FTT_LAUNCHED(ctx);
    op->max_segs = ceil_div(nnz, SEG) + nA;
    owned_free(ctx, cnt);
    owned_free(ctx, btot);
  }
  // entries in, two sorts of 12 B records, CSR + CSC records out
  prof_end(ctx, pb, PT_SCATTER, (double)nnz * (32.0 + 2 * 24.0 + 24.0 + 24.0), 0.0);
  owned_free(ctx, ra);
  owned_free(ctx, ca);
  owned_free(ctx, key_r);
  owned_free(ctx, key_c);
  owned_free(ctx, ident);
  owned_free(ctx, perm);
  owned_free(ctx, sorted);
  return FTT_OK;
}

void sparse_operand_free(ftt_ctx *ctx, SparseOperand *op) {
  owned_free(ctx, op->rptr);
  owned_free(ctx, op->cptr);
  owned_free(ctx, op->cidx_r);
  owned_free(ctx, op->v_r);
  owned_free(ctx, op->keyc);
  owned_free(ctx, op->v_c);
  owned_free(ctx, op->ridx_c);
  owned_free(ctx, op->cidx_c);
  owned_free(ctx, op->seg_base);
  owned_free(ctx, op->Qr);
  *op = SparseOperand();
}

int sparse_sketch(ftt_ctx *ctx, const SparseOperand &op, int64_t k, double *Y) {
  if (k > 64) {
    set_error("sparse sketch: k > 64");
    return FTT_ERR_INVALID;
  }
  double *Or = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&Or, 8 * (size_t)op.nA * k));
  k_omega_rows<<<grid_for(op.nA * k, 256, 4), 256, 0, ctx->stream>>>(op.nA, (int)k, Or);
  FTT_LAUNCHED(ctx);
  const int pb = prof_begin(ctx);
  k_spmm_rows<<<grid_for(op.mA, 8, 1, 148 * 32), 256, 0, ctx->stream>>>(op.mA, (int)k, op.rptr,
                                                                        op.cidx_r, op.v_r, Or, Y);
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb, PT_GEMM, 12.0 * op.nnz + 8.0 * op.mA * k, 2.0 * op.nnz * k);
  owned_free(ctx, Or);
  return FTT_OK;
}

int sparse_qt_a(ftt_ctx *ctx, SparseOperand &op, int64_t kr, const double *Q, double *B) {
  if (kr > 64) {
    set_error("sparse Q^T A: rank > 64");
    return FTT_ERR_INVALID;
  }
  // Q row-major (kept for the residual's entry term)
  owned_free(ctx, op.Qr);
  op.Qr = nullptr;
  op.ldq = (kr + 1) & ~(int64_t)1;  // even row stride: 16-byte aligned double2 rows
  FTT_CHECK(owned_alloc(ctx, (void **)&op.Qr, 8 * (size_t)op.mA * op.ldq));
  if (op.ldq != kr)
    FTT_CUDA(cudaMemsetAsync(op.Qr, 0, 8 * (size_t)op.mA * op.ldq, ctx->stream));
  FTT_CHECK(transpose(ctx, op.mA, kr, Q, op.mA, op.Qr, op.ldq));
  double *part = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&part, 8 * (size_t)op.max_segs * kr));
  const int pb = prof_begin(ctx);
  const int grid = grid_for(op.max_segs, 8, 1, 148 * 32);
#define FTT_SPB(KR_)                                                                              \
  k_spmm_seg<KR_><<<grid, 256, 0, ctx->stream>>>(op.nA, (int)kr, (int)op.ldq, op.max_segs, op.cptr,  \
                                                 op.seg_base,                                    \
                                                 op.ridx_c, op.v_c, op.Qr, part)
  if (kr <= 8) FTT_SPB(8);
  else if (kr <= 16) FTT_SPB(16);
  else if (kr <= 32) FTT_SPB(32);
  else FTT_SPB(64);
#undef FTT_SPB
  FTT_LAUNCHED(ctx);
  k_seg_reduce<<<grid_for(op.nA * kr, 256, 4), 256, 0, ctx->stream>>>(op.nA, (int)kr, op.seg_base,
                                                                      part, B);
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb, PT_GEMM, 12.0 * op.nnz + 8.0 * op.nA * kr, 2.0 * op.nnz * kr);
  owned_free(ctx, part);
  return FTT_OK;
}

int sparse_resid(ftt_ctx *ctx, SparseOperand &op, int64_t kr, const double *Q, const double *B,
                 double *out_dev) {
  if (kr > 64 || !op.Qr) {
    set_error("sparse residual: rank > 64 or no B");
    return FTT_ERR_INVALID;
  }
  const int64_t ncb = ceil_div(op.nA, 32);
  const int64_t wpr = ncb;  // bitmap words per row
  unsigned *bm = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&bm, 4 * (size_t)op.mA * wpr));
  FTT_CUDA(cudaMemsetAsync(bm, 0, 4 * (size_t)op.mA * wpr, ctx->stream));
  k_sp_bitmap<<<grid_for(op.nnz, 256, 4), 256, 0, ctx->stream>>>(op.nnz, op.ridx_c, op.cidx_c, wpr,
                                                                 bm);
  FTT_LAUNCHED(ctx);
  const int64_t ngx = ceil_div(op.nA, RCB);
  const int64_t want = std::max<int64_t>(1, ceil_div(8 * (int64_t)ctx->num_sms, ngx));
  const int64_t chunk = std::max<int64_t>(512, ceil_div(ceil_div(op.mA, want), 512) * 512);
  const int64_t nch = ceil_div(op.mA, chunk);
  const int64_t per = 8192;
  const int64_t non = ceil_div(op.nnz, per);
  if (ngx > 0x7fffffff || nch > 65535) {
    set_error("sparse residual: grid too large");
    return FTT_ERR_INVALID;
  }
  const int64_t noff = ngx * nch;
  double *part = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&part, 8 * (size_t)(noff + non)));
  dim3 grid((unsigned)ngx, (unsigned)nch);
  const int pb = prof_begin(ctx);
#define FTT_SPR(KR_, C_)                                                                         \
  do {                                                                                           \
    k_sp_resid_off<KR_, C_><<<grid, 256, 0, ctx->stream>>>(op.mA, op.nA, (int)kr, (int)op.ldq,   \
                                                           op.Qr, B, bm,                         \
                                                           wpr, chunk, part);                    \
    k_sp_resid_on<KR_><<<(unsigned)non, 256, 0, ctx->stream>>>(op.nnz, (int)kr, (int)op.ldq,     \
                                                               op.ridx_c,                        \
                                                               op.cidx_c, op.v_c, op.Qr, B, per,  \
                                                               part + noff);                     \
  } while (0)
  if (kr <= 8) FTT_SPR(8, 2);
  else if (kr <= 16) FTT_SPR(16, 2);
  else if (kr <= 32) FTT_SPR(32, 1);
  else FTT_SPR(64, 1);
#undef FTT_SPR
  FTT_LAUNCHED(ctx);
  // bitmap (written + read) + Q once per column group + entries; every
  // element of Q B formed once (2 kr flops)
  prof_end(ctx, pb, PT_GEMM, 8.0 * op.mA * wpr + 8.0 * op.mA * kr * ngx + 24.0 * op.nnz,
           2.0 * (double)op.mA * op.nA * kr);
  k_sp_sum<<<1, 1024, 0, ctx->stream>>>(part, noff + non, out_dev);
  FTT_LAUNCHED(ctx);
  owned_free(ctx, part);
  owned_free(ctx, bm);
  return FTT_OK;
}

}  // namespace ftt

// ---------------------------------------------------------------------------
// depar_general (fasttt.py:96-145): the floating-point deparallelisation.
// Columns are visited in order (first-occurrence classes, as the
// reference's loop); for column u the kept basis columns b_i are tested in
// parallel (one warp per basis column): coeff_i = (b_i . u) / |b_i|^2, the
// residual |u - coeff_i b_i|^2 evaluated explicitly, hit_i = rnorm2 <= tol^2
// |u|^2; the lowest hit index wins, else u joins the basis.  One CTA walks the
// columns (the kept set depends on every earlier decision).
namespace ftt {
namespace {

__global__ void __launch_bounds__(1024) k_depar_general(int64_t rows, int64_t cols,
                                                        const double *__restrict__ M, int64_t ldm,
                                                        double tol, int64_t *__restrict__ kept,
                                                        double *__restrict__ bnorm2,
                                                        int64_t *__restrict__ t_row,
                                                        double *__restrict__ t_coeff,
                                                        int64_t *__restrict__ width_at,
                                                        int64_t *__restrict__ width_out) {
  __shared__ double red[32];
  __shared__ int s_hit;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  int64_t width = 0;
  for (int64_t j = 0; j < cols; ++j) {
    const double *u = M + j * ldm;
    double a = 0.0;
    for (int64_t r = tid; r < rows; r += blockDim.x) a += u[r] * u[r];
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) red[warp] = a;
    if (tid == 0) s_hit = 0x7fffffff;
    __syncthreads();
    double unorm2 = 0.0;
    for (int w = 0; w < nw; ++w) unorm2 += red[w];
    if (tid == 0) width_at[j] = width;
    if (unorm2 == 0.0) {
      if (tid == 0) {
        t_row[j] = -1;
        t_coeff[j] = 0.0;
      }
      __syncthreads();
      continue;
    }
    const double thr = tol * tol * unorm2;
    for (int64_t i = warp; i < width; i += nw) {
      const double *b = M + kept[i] * ldm;
      double dot = 0.0;
      for (int64_t r = lane; r < rows; r += 32) dot += b[r] * u[r];
      for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      const double coeff = dot / bnorm2[i];
      double rn = 0.0;
      for (int64_t r = lane; r < rows; r += 32) {
        const double e = u[r] - b[r] * coeff;
        rn += e * e;
      }
      for (int o = 16; o; o >>= 1) rn += __shfl_xor_sync(0xffffffffu, rn, o);
      if (lane == 0 && rn <= thr) atomicMin(&s_hit, (int)i);
      (void)coeff;
    }
    __syncthreads();
    const int hit = s_hit;
    if (hit != 0x7fffffff) {
      // the winner's coefficient (recomputed by one warp: same arithmetic)
      if (warp == 0) {
        const double *b = M + kept[hit] * ldm;
        double dot = 0.0;
        for (int64_t r = lane; r < rows; r += 32) dot += b[r] * u[r];
        for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (lane == 0) {
          t_row[j] = hit;
          t_coeff[j] = dot / bnorm2[hit];
        }
      }
    } else if (tid == 0) {
      kept[width] = j;
      bnorm2[width] = unorm2;
      t_row[j] = width;
      t_coeff[j] = 1.0;
    }
    if (hit == 0x7fffffff) ++width;
    __syncthreads();
  }
  if (tid == 0) *width_out = width;
}

}  // namespace
}  // namespace ftt

using namespace ftt;

extern "C" int ftt_depar_general(ftt_ctx *ctx, int64_t rows, int64_t cols, const double *M,
                                 int64_t ldm, double tol, int64_t *kept, int64_t *t_row,
                                 double *t_coeff, int64_t *width_at, int64_t *width_out) {
  if (!ctx || rows < 0 || cols < 0 || !width_out || ldm < std::max<int64_t>(rows, 1) || tol < 0) {
    set_error("ftt_depar_general: invalid arguments");
    return FTT_ERR_INVALID;
  }
  *width_out = 0;
  if (cols == 0) return FTT_OK;
  double *bn = nullptr;
  int64_t *wdev = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&bn, 8 * (size_t)cols));
  FTT_CHECK(owned_alloc(ctx, (void **)&wdev, 64));
  k_depar_general<<<1, 1024, 0, ctx->stream>>>(rows, cols, M, ldm, tol, kept, bn, t_row, t_coeff,
                                               width_at, wdev);
  FTT_LAUNCHED(ctx);
  FTT_CHECK(copy_to_host(ctx, width_out, wdev, sizeof(int64_t)));
  owned_free(ctx, bn);
  owned_free(ctx, wdev);
  return FTT_OK;
}
