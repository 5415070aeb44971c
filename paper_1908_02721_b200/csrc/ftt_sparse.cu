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
    if (key_r) key_r[e] = (uint64_t)r;
    key_c[e] = (uint64_t)c;  // stable sort by column keeps rows ascending (see below)
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

// The sparse operand's test matrix is a sign matrix (Rademacher sketch):
// Omega[c, j] = +1 / -1 by bit j of splitmix64(c), one 64-bit word per
// column c of A_tall (k <= 64).  The dense path streams a uniform [-1, 1)
// Omega through a GEMM; here every entry of A would fetch its k-double row of
// Omega from L2 (config 5: 8.5 M x 256 B, the whole cost of the sketch),
// while the sign words of all columns stay in L1 and the product is one add
// per entry and sketch column.  The certificate (section 4a) judges the
// basis either way.
__global__ void k_omega_bits(int64_t nA, uint64_t *__restrict__ Ob) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nA;
       c += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)c + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    Ob[c] = z;
  }
}

// Fiber-level CSR of the transposed operand (rows of A_tall = s_map values):
// the key of fiber f is its row; a stable sort of the R fibers by that key
// replaces the sort of the nnz entries -- a row's entries are its fibers'
// (ascending fiber, then the fiber's own entries), the order the entry-level
// CSR holds them in.
__global__ void k_sp_fiber_keys(int64_t R, const int64_t *__restrict__ smap,
                                uint64_t *__restrict__ key, uint32_t *__restrict__ ident) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < R;
       f += (int64_t)gridDim.x * blockDim.x) {
    key[f] = (uint64_t)smap[f];
    ident[f] = (uint32_t)f;
  }
}

// The sorted fibers' entry ranges and column blocks, gathered once so that
// the sketch kernel reads them with the row's fiber list (one load round).
__global__ void k_sp_fiber_desc(int64_t R, const uint32_t *__restrict__ fperm,
                                const int64_t *__restrict__ indptr,
                                const int64_t *__restrict__ tmap, int64_t np,
                                int64_t *__restrict__ fe0, int32_t *__restrict__ flen,
                                int32_t *__restrict__ fcb) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < R;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = fperm[j];
    const int64_t e0 = indptr[f];
    fe0[j] = e0;
    flen[j] = (int32_t)(indptr[f + 1] - e0);
    fcb[j] = (int32_t)((tmap ? tmap[f] : 0) * np);
  }
}

// Y = A_tall Omega on the fiber-level CSR: one warp per row.  The lanes take
// up to 32 of the row's fibers at once (entry range and column block), a warp
// scan lays their entries out in slots, each lane writes its fiber's (column,
// value) pairs into the warp's shared slots, and the warp then accumulates
// the slots in order -- the same sequence of additions as k_spmm_rows on the
// entry-level CSR (bit-identical Y).  The next row's offsets and fiber
// descriptors are fetched while the current row is accumulated, so one
// dependent load round (the entries) is exposed per row instead of four.
constexpr int SPF_SLOTS = 128;

__global__ void __launch_bounds__(256) k_spmm_rows_f(int64_t mA, int k,
                                                     const int64_t *__restrict__ rptr,
                                                     const int64_t *__restrict__ fe0,
                                                     const int32_t *__restrict__ flen,
                                                     const int32_t *__restrict__ fcb,
                                                     const int64_t *__restrict__ pidx,
                                                     const double *__restrict__ vals,
                                                     const uint64_t *__restrict__ Ob,
                                                     double *__restrict__ Y) {
  __shared__ int32_t s_col[8][SPF_SLOTS];
  __shared__ double s_w[8][SPF_SLOTS];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned full = 0xffffffffu;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + wid;
  if (r >= mA) return;
  // software pipeline: (j0, j1) of row r + 2 warps and the first batch's
  // descriptors of row r + warps are in flight while row r is accumulated
  int64_t j0 = rptr[r], j1 = rptr[r + 1];
  int64_t e0 = 0;
  int len = 0, cb = 0;
  if (j0 + lane < j1) {
    e0 = fe0[j0 + lane];
    len = flen[j0 + lane];
    cb = fcb[j0 + lane];
  }
  int64_t rn = r + warps, j0n = 0, j1n = 0;
  if (rn < mA) {
    j0n = rptr[rn];
    j1n = rptr[rn + 1];
  }
  for (; r < mA;) {
    const int64_t rnn = rn + warps;
    int64_t j0nn = 0, j1nn = 0;
    if (rnn < mA) {
      j0nn = rptr[rnn];
      j1nn = rptr[rnn + 1];
    }
    int64_t e0n = 0;
    int lenn = 0, cbn = 0;
    if (rn < mA && j0n + lane < j1n) {
      e0n = fe0[j0n + lane];
      lenn = flen[j0n + lane];
      cbn = fcb[j0n + lane];
    }
    double a0 = 0.0, a1 = 0.0;
    auto add = [&](int64_t c, double w) {
      const uint64_t bits = __ldg(Ob + c);
      a0 += (bits >> lane) & 1 ? w : -w;
      a1 += (bits >> (lane + 32)) & 1 ? w : -w;
    };
    bool first = true;
    for (int64_t jb = j0; jb < j1;) {
      const int nf = (int)min((int64_t)32, j1 - jb);
      if (!first) {  // rows with more than one batch: fetched in place
        e0 = 0;
        len = 0;
        cb = 0;
        if (lane < nf) {
          e0 = fe0[jb + lane];
          len = flen[jb + lane];
          cb = fcb[jb + lane];
        }
      }
      first = false;
      int cum = len;  // inclusive scan of the fibers' lengths
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(full, cum, o);
        if (lane >= o) cum += t;
      }
      // this round: the leading fibers whose entries fit the slots
      const int take = __popc(__ballot_sync(full, lane < nf && cum <= SPF_SLOTS));
      if (take == 0) {  // a fiber longer than the slots: straight from global
        const int64_t fe = __shfl_sync(full, e0, 0);
        const int fc = __shfl_sync(full, cb, 0), fl = __shfl_sync(full, len, 0);
        for (int t = 0; t < fl; ++t) add(fc + pidx[fe + t], vals[fe + t]);
        jb += 1;
        first = false;
        // (the remaining lanes' descriptors are refetched: batch start moved)
        continue;
      }
      const int total = __shfl_sync(full, cum, take - 1);
      if (lane < take) {
        const int base = cum - len;
        for (int t = 0; t < len; ++t) {
          s_col[wid][base + t] = (int32_t)(cb + pidx[e0 + t]);
          s_w[wid][base + t] = vals[e0 + t];
        }
      }
      __syncwarp();
      for (int u = 0; u < total; ++u) add(s_col[wid][u], s_w[wid][u]);
      __syncwarp();
      jb += take;
    }
    if (lane < k) Y[r + (int64_t)lane * mA] = a0;
    if (lane + 32 < k) Y[r + (int64_t)(lane + 32) * mA] = a1;
    r = rn;
    j0 = j0n;
    j1 = j1n;
    e0 = e0n;
    len = lenn;
    cb = cbn;
    rn = rnn;
    j0n = j0nn;
    j1n = j1nn;
  }
}

// Y = A_tall Omega (mA x k col-major): one warp per row, lanes j and j + 32.
__global__ void __launch_bounds__(256) k_spmm_rows(int64_t mA, int k, const int64_t *__restrict__ rptr,
                                                   const int32_t *__restrict__ cidx,
                                                   const double *__restrict__ v,
                                                   const uint64_t *__restrict__ Ob,
                                                   double *__restrict__ Y) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < mA; r += warps) {
    const int64_t e0 = rptr[r], e1 = rptr[r + 1];
    double a0 = 0.0, a1 = 0.0;
    int64_t e = e0;
    for (; e + 4 <= e1; e += 4) {  // four entries' loads in flight together
      int32_t c[4];
      double w[4];
      uint64_t b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] = cidx[e + u];
        w[u] = v[e + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = __ldg(Ob + c[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0 += (b[u] >> lane) & 1 ? w[u] : -w[u];
        a1 += (b[u] >> (lane + 32)) & 1 ? w[u] : -w[u];
      }
    }
    for (; e < e1; ++e) {
      const uint64_t b = __ldg(Ob + cidx[e]);
      const double w = v[e];
      a0 += (b >> lane) & 1 ? w : -w;
      a1 += (b >> (lane + 32)) & 1 ? w : -w;
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

// ---- residual energy rest2 = ||A - Q B||_F^2 in double-double ------------
// rest2 = S2 + S1 with S2 = sum over the entries of (A_rc - (QB)_rc)^2 (a sum
// of small nonnegative terms, plain fp64) and S1 = sum over the positions
// WITHOUT an entry of (QB)_rc^2, evaluated as
//     S1 = sum_c b_c^T G b_c - sum_entries (QB)_rc^2,   G = Q^T Q,
// where both sums are ~||A||^2 and S1 is ~eps^2 ||A||^2: every term is
// carried in double-double (~2^-104 relative, pairwise/blocked sums), so the
// difference keeps ~1e-30 ||A||^2 absolute accuracy -- far below the
// certificate's 1e-6 delta^2 resolution -- without forming the m x n matrix
// Q B (the fp64 direct sum over all m n positions it replaces cost ~2.5 ms
// on config 5; this is O(m kr^2 + nnz kr)).
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd dd_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_fast(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd dd_add(dd x, dd y) {
  dd s = dd_two_sum(x.hi, y.hi);
  s.lo += x.lo + y.lo;
  return dd_fast(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_prod(double a, double b) {  // exact a * b
  const double p = a * b;
  return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd dd_mul(dd x, dd y) {
  const double p = x.hi * y.hi;
  const double e = fma(x.hi, y.hi, -p) + (x.hi * y.lo + x.lo * y.hi);
  return dd_fast(p, e);
}
__device__ __forceinline__ dd dd_shfl_down(dd x, int o) {
  return {__shfl_down_sync(0xffffffffu, x.hi, o), __shfl_down_sync(0xffffffffu, x.lo, o)};
}

// Partial Gram G = Q^T Q (row-major Q, ldq) in double-double: block b sums
// rows [b * per, (b + 1) * per) staged in shared memory in ROWS-row tiles;
// thread t owns the pairs (a, c) = t, t + 256, ... of the KR x KR matrix.
template <int KR>
__global__ void __launch_bounds__(256) k_gram_dd(int64_t mA, int kr, int ldq,
                                                 const double *__restrict__ Qr, int64_t per,
                                                 dd *__restrict__ part) {
  constexpr int ROWS = 4096 / KR;
  constexpr int PAIRS = (KR * KR + 255) / 256;
  __shared__ __align__(16) double Qs[ROWS][KR];
  dd acc[PAIRS];
#pragma unroll
  for (int q = 0; q < PAIRS; ++q) acc[q] = {0.0, 0.0};
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(mA, r0 + per);
  for (int64_t base = r0; base < r1; base += ROWS) {
    const int nr = (int)min((int64_t)ROWS, r1 - base);
    __syncthreads();
    for (int e = threadIdx.x; e < ROWS * KR; e += 256) {
      const int rr = e / KR, j = e - rr * KR;
      Qs[rr][j] = (rr < nr && j < kr) ? Qr[(base + rr) * ldq + j] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PAIRS; ++q) {
      const int pr = threadIdx.x + 256 * q;
      if (pr < KR * KR) {
        const int a = pr / KR, c = pr - a * KR;
        dd s = acc[q];
        for (int rr = 0; rr < nr; ++rr) s = dd_add(s, dd_prod(Qs[rr][a], Qs[rr][c]));
        acc[q] = s;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < PAIRS; ++q) {
    const int pr = threadIdx.x + 256 * q;
    if (pr < KR * KR) part[(int64_t)blockIdx.x * KR * KR + pr] = acc[q];
  }
}

// G = fixed-order sum of the block partials (one thread per pair).
__global__ void k_gram_reduce_dd(int pairs, int64_t nparts, const dd *__restrict__ part,
                                 dd *__restrict__ G) {
  const int pr = blockIdx.x * blockDim.x + threadIdx.x;
  if (pr >= pairs) return;
  dd s = {0.0, 0.0};
  for (int64_t b = 0; b < nparts; ++b) s = dd_add(s, part[b * pairs + pr]);
  G[pr] = s;
}

// sum over the columns c of B (kr x nA, column-major) of b_c^T G b_c in dd:
// columns striped over the threads of the grid, a fixed-order tree per
// block; out[blockIdx.x] = the block's partial.
template <int KR>
__global__ void __launch_bounds__(256) k_gram_form_dd(int64_t nA, int kr,
                                                      const dd *__restrict__ G,
                                                      const double *__restrict__ B,
                                                      dd *__restrict__ out) {
  __shared__ dd red[256];
  dd tot = {0.0, 0.0};
  for (int64_t c = blockIdx.x * 256 + threadIdx.x; c < nA; c += 256 * (int64_t)gridDim.x) {
    const double *bc = B + c * kr;
    dd col = {0.0, 0.0};
    for (int a = 0; a < kr; ++a) {
      for (int e = 0; e < kr; ++e) {
        const dd w = dd_prod(bc[a], bc[e]);
        col = dd_add(col, dd_mul(w, G[a * KR + e]));
      }
    }
    tot = dd_add(tot, col);
  }
  red[threadIdx.x] = tot;
  __syncthreads();
  for (int off = 128; off; off >>= 1) {
    if ((int)threadIdx.x < off) red[threadIdx.x] = dd_add(red[threadIdx.x], red[threadIdx.x + off]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = red[0];
}

// Over the entries (CSC arrays, a fixed range per block): (QB)_rc in dd, its
// square summed in dd (S_on), and (A_rc - (QB)_rc)^2 summed in fp64 (S2).
template <int KR>
__global__ void __launch_bounds__(256) k_sp_on_dd(int64_t nnz, int kr, int ldq,
                                                  const int32_t *__restrict__ ridx,
                                                  const int32_t *__restrict__ cidx,
                                                  const double *__restrict__ v,
                                                  const double *__restrict__ Qr,
                                                  const double *__restrict__ B, int64_t per,
                                                  dd *__restrict__ part_on,
                                                  double *__restrict__ part_s2) {
  __shared__ dd red1[8];
  __shared__ double red2[8];
  const int64_t e0 = (int64_t)blockIdx.x * per, e1 = min(nnz, e0 + per);
  dd on = {0.0, 0.0};
  double s2 = 0.0;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const double2 *q = reinterpret_cast<const double2 *>(Qr + (int64_t)ridx[e] * ldq);
    const double *bc = B + (int64_t)cidx[e] * kr;
    dd qb = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < KR; j += 2)
      if (j < kr) {
        const double2 t = __ldg(q + j / 2);
        qb = dd_add(qb, dd_prod(t.x, bc[j]));
        if (j + 1 < kr) qb = dd_add(qb, dd_prod(t.y, bc[j + 1]));
      }
    on = dd_add(on, dd_mul(qb, qb));
    const double d = (v[e] - qb.hi) - qb.lo;
    s2 += d * d;
  }
  for (int o = 16; o; o >>= 1) {
    on = dd_add(on, dd_shfl_down(on, o));
    s2 += __shfl_down_sync(0xffffffffu, s2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red1[threadIdx.x >> 5] = on;
    red2[threadIdx.x >> 5] = s2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    dd a = {0.0, 0.0};
    double b = 0.0;
    for (int i = 0; i < 8; ++i) {
      a = dd_add(a, red1[i]);
      b += red2[i];
    }
    part_on[blockIdx.x] = a;
    part_s2[blockIdx.x] = b;
  }
}

// rest2 = S2 + (S_all - S_on), the block partials summed in fixed order.
__global__ void __launch_bounds__(256) k_resid_combine(int64_t n, const dd *__restrict__ part_on,
                                                       const double *__restrict__ part_s2,
                                                       int nall, const dd *__restrict__ s_all,
                                                       double *__restrict__ out) {
  __shared__ dd r1[256];
  __shared__ double r2[256];
  __shared__ dd all;
  if (threadIdx.x == 0) {
    dd t = {0.0, 0.0};
    for (int i = 0; i < nall; ++i) t = dd_add(t, s_all[i]);
    all = t;
  }
  dd a = {0.0, 0.0};
  double b = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) {
    a = dd_add(a, part_on[i]);
    b += part_s2[i];
  }
  r1[threadIdx.x] = a;
  r2[threadIdx.x] = b;
  __syncthreads();
  for (int off = 128; off; off >>= 1) {
    if ((int)threadIdx.x < off) {
      r1[threadIdx.x] = dd_add(r1[threadIdx.x], r1[threadIdx.x + off]);
      r2[threadIdx.x] += r2[threadIdx.x + off];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const dd neg = {-r1[0].hi, -r1[0].lo};
    const dd s1 = dd_add(all, neg);
    *out = r2[0] + fmax(s1.hi + s1.lo, 0.0);
  }
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
                         const int64_t *smap, int64_t np, int64_t m, int64_t n, int64_t R,
                         const int64_t *indptr) {
  op->nnz = nnz;
  op->transposed = m < n;
  op->mA = std::max(m, n);
  op->nA = std::min(m, n);
  const int64_t mA = op->mA, nA = op->nA;
  // rows of the transposed operand are s_map values: CSR at fiber level
  op->by_fiber = op->transposed && indptr && R > 0 && smap;
  op->f_indptr = indptr;
  op->f_pidx = pidx;
  op->f_vals = vals;
  op->f_tmap = tmap;
  op->f_np = np;
  const bool by_fiber = op->by_fiber;
  int32_t *ra = nullptr, *ca = nullptr;
  uint64_t *key_r = nullptr, *key_c = nullptr, *sorted = nullptr;
  uint32_t *ident = nullptr, *perm = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&ra, 4 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&ca, 4 * (size_t)nnz));
  if (!by_fiber) FTT_CHECK(owned_alloc(ctx, (void **)&key_r, 8 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&key_c, 8 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&ident, 4 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&perm, 4 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->rptr, 8 * (size_t)(mA + 1)));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->cptr, 8 * (size_t)(nA + 1)));
  if (!by_fiber) {
    FTT_CHECK(owned_alloc(ctx, (void **)&op->cidx_r, 4 * (size_t)nnz));
    FTT_CHECK(owned_alloc(ctx, (void **)&op->v_r, 8 * (size_t)nnz));
  }
  FTT_CHECK(owned_alloc(ctx, (void **)&op->keyc, 8 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->v_c, 8 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->ridx_c, 4 * (size_t)nnz));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->cidx_c, 4 * (size_t)nnz));
  const int pb = prof_begin(ctx);
  k_sp_entries<<<grid_for(nnz, 256, 4), 256, 0, ctx->stream>>>(
      nnz, fiber_of, pidx, tmap, smap, np, op->transposed ? 1 : 0, mA, ra, ca, key_r, key_c, ident);
  FTT_LAUNCHED(ctx);
  if (by_fiber) {
    // CSR over the R fibers: stable sort by row, a row's fibers stay ascending
    uint64_t *kf = nullptr;
    uint32_t *idf = nullptr;
    FTT_CHECK(owned_alloc(ctx, (void **)&kf, 8 * (size_t)R));
    FTT_CHECK(owned_alloc(ctx, (void **)&idf, 4 * (size_t)R));
    FTT_CHECK(owned_alloc(ctx, (void **)&sorted, 8 * (size_t)R));
    FTT_CHECK(owned_alloc(ctx, (void **)&op->fperm, 4 * (size_t)R));
    k_sp_fiber_keys<<<grid_for(R, 256, 4), 256, 0, ctx->stream>>>(R, smap, kf, idf);
    FTT_LAUNCHED(ctx);
    FTT_CHECK(arena_reserve(ctx, radix_sort_scratch_bytes(R, true) + 4096));
    FTT_CHECK(radix_sort(ctx, kf, idf, sorted, op->fperm, R, bits_for((uint64_t)(mA - 1))));
    k_lower_bounds<<<grid_for(mA + 1, 256, 4), 256, 0, ctx->stream>>>(sorted, R, mA, 1, op->rptr);
    FTT_LAUNCHED(ctx);
    FTT_CHECK(owned_alloc(ctx, (void **)&op->fe0, 8 * (size_t)R));
    FTT_CHECK(owned_alloc(ctx, (void **)&op->flen, 4 * (size_t)R));
    FTT_CHECK(owned_alloc(ctx, (void **)&op->fcb, 4 * (size_t)R));
    k_sp_fiber_desc<<<grid_for(R, 256, 4), 256, 0, ctx->stream>>>(R, op->fperm, indptr, tmap, np,
                                                                  op->fe0, op->flen, op->fcb);
    FTT_LAUNCHED(ctx);
    owned_free(ctx, kf);
    owned_free(ctx, idf);
  } else {
    // CSR: stable sort by row (entries of a row keep the fiber order)
    FTT_CHECK(arena_reserve(ctx, radix_sort_scratch_bytes(nnz, true) + 4096));
    FTT_CHECK(owned_alloc(ctx, (void **)&sorted, 8 * (size_t)nnz));
    FTT_CHECK(radix_sort(ctx, key_r, ident, sorted, perm, nnz, bits_for((uint64_t)(mA - 1))));
    k_lower_bounds<<<grid_for(mA + 1, 256, 4), 256, 0, ctx->stream>>>(sorted, nnz, mA, 1, op->rptr);
    FTT_LAUNCHED(ctx);
    k_sp_gather<<<grid_for(nnz, 256, 4), 256, 0, ctx->stream>>>(nnz, perm, ca, vals, op->cidx_r,
                                                                 op->v_r);
    FTT_LAUNCHED(ctx);
  }
  // CSC: a STABLE sort by column alone.  In fiber order (fibers by
  // (prefix, suffix), nonzeros by pivot index) the entries sharing a column
  // of A_tall already come with ascending rows -- t_map is monotone in the
  // prefix and s_map in the suffix -- so (column, row) order needs only the
  // column's bits (config 5: 13 bits, 2 passes instead of 4).
  FTT_CHECK(arena_reserve(ctx, radix_sort_scratch_bytes(nnz, true) + 4096));
  FTT_CHECK(radix_sort(ctx, key_c, ident, op->keyc, perm, nnz, bits_for((uint64_t)(nA - 1))));
  k_lower_bounds<<<grid_for(nA + 1, 256, 4), 256, 0, ctx->stream>>>(op->keyc, nnz, nA, 1,
                                                                     op->cptr);
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
  owned_free(ctx, op->fperm);
  owned_free(ctx, op->fe0);
  owned_free(ctx, op->flen);
  owned_free(ctx, op->fcb);
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
  uint64_t *Or = nullptr;  // sign words of Omega's rows
  FTT_CHECK(owned_alloc(ctx, (void **)&Or, 8 * (size_t)op.nA));
  k_omega_bits<<<grid_for(op.nA, 256, 4), 256, 0, ctx->stream>>>(op.nA, Or);
  FTT_LAUNCHED(ctx);
  const int pb = prof_begin(ctx);
  if (op.by_fiber)
    k_spmm_rows_f<<<grid_for(op.mA, 8, 1, 148 * 32), 256, 0, ctx->stream>>>(
        op.mA, (int)k, op.rptr, op.fe0, op.flen, op.fcb, op.f_pidx, op.f_vals, Or, Y);
  else
    k_spmm_rows<<<grid_for(op.mA, 8, 1, 148 * 32), 256, 0, ctx->stream>>>(op.mA, (int)k, op.rptr,
                                                                          op.cidx_r, op.v_r, Or, Y);
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb, PT_GEMM, 12.0 * op.nnz + 8.0 * op.mA * k, 1.0 * op.nnz * k);
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
  (void)Q;  // the row-major copy op.Qr (from sparse_qt_a) is what the kernels read
  if (kr > 64 || !op.Qr) {
    set_error("sparse residual: rank > 64 or no B");
    return FTT_ERR_INVALID;
  }
  const int64_t ngram = std::min<int64_t>(2 * (int64_t)ctx->num_sms, std::max<int64_t>(1, ceil_div(op.mA, 256)));
  const int64_t per_g = ceil_div(op.mA, ngram);
  const int64_t per = 8192;
  const int64_t non = ceil_div(op.nnz, per);
  const int kk = kr <= 8 ? 8 : kr <= 16 ? 16 : kr <= 32 ? 32 : 64;
  char *buf = nullptr;
  const size_t b_gram = align_up(sizeof(dd) * (size_t)ngram * kk * kk);
  const size_t b_on = align_up(sizeof(dd) * (size_t)std::max<int64_t>(non, 1));
  const size_t b_s2 = align_up(sizeof(double) * (size_t)std::max<int64_t>(non, 1));
  const size_t b_g = align_up(sizeof(dd) * (size_t)kk * kk);
  const int nform = (int)std::min<int64_t>(ctx->num_sms, std::max<int64_t>(1, ceil_div(op.nA, 256)));
  FTT_CHECK(owned_alloc(ctx, (void **)&buf, b_gram + b_on + b_s2 + b_g + align_up(sizeof(dd) * nform)));
  dd *gpart = reinterpret_cast<dd *>(buf);
  dd *on = reinterpret_cast<dd *>(buf + b_gram);
  double *s2 = reinterpret_cast<double *>(buf + b_gram + b_on);
  dd *G = reinterpret_cast<dd *>(buf + b_gram + b_on + b_s2);
  dd *sall = reinterpret_cast<dd *>(buf + b_gram + b_on + b_s2 + b_g);
  const int pb = prof_begin(ctx);
#define FTT_SPR(KR_)                                                                              \
  do {                                                                                            \
    k_gram_dd<KR_><<<(unsigned)ngram, 256, 0, ctx->stream>>>(op.mA, (int)kr, (int)op.ldq, op.Qr,  \
                                                             per_g, gpart);                        \
    k_gram_reduce_dd<<<(KR_ * KR_ + 255) / 256, 256, 0, ctx->stream>>>(KR_ * KR_, ngram, gpart, G); \
    k_gram_form_dd<KR_><<<nform, 256, 0, ctx->stream>>>(op.nA, (int)kr, G, B, sall);             \
    k_sp_on_dd<KR_><<<(unsigned)std::max<int64_t>(non, 1), 256, 0, ctx->stream>>>(                \
        op.nnz, (int)kr, (int)op.ldq, op.ridx_c, op.cidx_c, op.v_c, op.Qr, B, per, on, s2);      \
  } while (0)
  if (kk == 8) FTT_SPR(8);
  else if (kk == 16) FTT_SPR(16);
  else if (kk == 32) FTT_SPR(32);
  else FTT_SPR(64);
#undef FTT_SPR
  FTT_LAUNCHED(ctx);
  k_resid_combine<<<1, 256, 0, ctx->stream>>>(std::max<int64_t>(non, 1), on, s2, nform, sall, out_dev);
  FTT_LAUNCHED(ctx);
  // Q read once (Gram), the entries (16 B) + a Q row and a B column per entry
  prof_end(ctx, pb, PT_GEMM, 8.0 * op.mA * kr + 16.0 * op.nnz, 2.0 * (double)op.mA * kr * kr +
                                                              2.0 * (double)op.nnz * kr);
  owned_free(ctx, buf);
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
