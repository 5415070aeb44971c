// fp64 GEMM on the B200 DMMA pipe (mma.sync.aligned.m8n8k4 .f64) with
// BLAS dgemm semantics (column-major, op = N/T).  Used for every dense core
// contraction of the rounding sweeps (fasttt.py:341, 347, 355) and inside
// the blocked Householder QR / Jacobi SVD.  tcgen05 has no f64 kind on
// sm_100a (ptxas rejects .kind::f64), so DMMA is the fp64 tensor path.
//
// CTA tile TBM x TBN x 16 (64x64 by default; 128 x {16,32,40,48} for narrow
// outputs, {16,32,48} x 128 for short ones, 16/32/48 squares for small ones), 4
// warps, k-tiles staged through an NSTAGE-deep cp.async ring in dynamic
// shared memory.  Split-K with a deterministic reduction when the output has
// too few tiles for 148 SMs.
#include "ftt_common.cuh"
#include "ftt_dense.cuh"

#include <vector>

namespace ftt {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, GT = 128;
constexpr int PAD = 4;  // (64+4) doubles = 136 words == 8 banks: conflict-free fragment loads

__device__ __forceinline__ int64_t ceil_div_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// EPI 0: C = alpha op(A) op(B) + beta C (or split-K partials).
// EPI 1: residual norm -- no C write; each CTA writes
//   npart[tile] = sum over its tile of (R0(row, col) - op(A) op(B))^2,
// R0 = C read-only, stored transposed when c_trans (R0(row, col) at
// C[col + row * ldc]).  Used by the certified low-rank SVD to form
// ||A - Q B||_F without materialising the residual.
// Tile TBM x TBN, 4 warps of (TBM/WM) x (TBN/WN) (MI x NJ DMMA 8x8 tiles),
// BK = 16, NSTAGE k-tiles in flight.
// Called by every thread after thread 0 wrote this CTA's npart entry: the
// last CTA of the grid to arrive (counter, reset by it) sums the nt
// partials in index order into *out (replaces a separate k_sum_partials).
__device__ __forceinline__ void last_cta_sum(const double *npart, int64_t nt, double *out,
                                             unsigned *counter) {
  __shared__ int s_last;
  __shared__ double s_w[32];
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned tk = atomicAdd(counter, 1u);
    s_last = tk == (unsigned)(nt - 1);
    if (s_last) *counter = 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < nt; i += blockDim.x) a += __ldcg(npart + i);
  for (int o = 16; o; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_w[w];
    *out = t;
  }
}

// cp.async (LDGSTS) helpers: 8-byte element copies with zero fill when
// `bytes` is 0 (out-of-range rows / columns / k), grouped per k-stage.
__device__ __forceinline__ void gm_cp8(double *smem, const double *gmem, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void gm_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void gm_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// k-stages in flight per CTA (the LDGSTS ring): the long-K Gram-type
// products (Q^T A over 10^5..3*10^5 rows) were latency bound at one
// register-prefetched stage (~1 TB/s); NSTAGE-1 stages ahead keep
// ~50-100 KB per SM in flight.
#ifndef FTT_GEMM_STAGES
#define FTT_GEMM_STAGES 4
#endif
constexpr int NSTAGE = FTT_GEMM_STAGES;
// warps along M for a TBM x TBN tile (4 warps per CTA)
__host__ __device__ constexpr int tile_wm(int tbm, int tbn) { return tbn == 128 ? 1 : (tbm == 128 ? 4 : 2); }
constexpr size_t gemm_smem_bytes(int tbm, int tbn) {
  return sizeof(double) * (size_t)NSTAGE * BK * ((tbm + PAD) + (tbn + PAD));
}

template <bool TA, bool TB, int EPI = 0, int TBM = 64, int TBN = 64>
__global__ void __launch_bounds__(GT) k_dgemm(int64_t m, int64_t n, int64_t k, double alpha,
                                              const double *__restrict__ A, int64_t lda,
                                              const double *__restrict__ B, int64_t ldb, double beta,
                                              double *__restrict__ C, int64_t ldc, int64_t kps,
                                              double *__restrict__ partial, int c_trans = 0,
                                              double *__restrict__ npart = nullptr,
                                              unsigned *__restrict__ tile_cnt = nullptr,
                                              double *__restrict__ sum_out = nullptr) {
  constexpr int WM = tile_wm(TBM, TBN);  // warps along M
  constexpr int WN = 4 / WM;             // warps along N
  constexpr int MI = TBM / WM / 8;       // 8x8 DMMA tiles per warp along M
  constexpr int NJ = TBN / WN / 8;       // ... along N
  constexpr int LA = TBM + PAD, LB = TBN + PAD;
  constexpr int RA = TBM * BK / GT;      // A-tile elements per thread
  constexpr int RB = TBN * BK / GT;      // B-tile elements per thread
  static_assert(WM * WN == 4 && MI * 8 * WM == TBM && NJ * 8 * WN == TBN, "tile shape");
  static_assert(RA * GT == TBM * BK && RB * GT == TBN * BK, "tile load split");
  static_assert(LA % 16 == 4 || LA % 16 == 12, "A row stride must be conflict-free");
  static_assert(LB % 16 == 4 || LB % 16 == 12, "B row stride must be conflict-free");
  extern __shared__ __align__(16) double gm_smem[];
  double *const As0 = gm_smem;                         // [NSTAGE][BK][LA]
  double *const Bs0 = gm_smem + (size_t)NSTAGE * BK * LA;  // [NSTAGE][BK][LB]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp % WM) * (MI * 8), wn = (warp / WM) * (NJ * 8);
  const int64_t tm = (int64_t)blockIdx.x * TBM, tn = (int64_t)blockIdx.y * TBN;
  const int64_t kb = (int64_t)blockIdx.z * kps;
  const int64_t ke = min(k, kb + kps);
  const int64_t nk = ke > kb ? (ke - kb + BK - 1) / BK : 0;

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // issue the copies of k-tile t into ring slot t % NSTAGE
  auto issue = [&](int64_t t) {
    const int slot = (int)(t % NSTAGE);
    const int64_t k0 = kb + t * BK;
    double *As = As0 + (size_t)slot * BK * LA;
    double *Bs = Bs0 + (size_t)slot * BK * LB;
#pragma unroll
    for (int r = 0; r < RA; ++r) {
      const int e = r * GT + tid;
      int i, kk;
      if (!TA) {
        i = e % TBM;
        kk = e / TBM;
      } else {
        kk = e % BK;
        i = e / BK;
      }
      const int64_t gi = tm + i, gk = k0 + kk;
      const bool ok = gi < m && gk < ke;
      gm_cp8(As + kk * LA + i, ok ? (TA ? A + gk + gi * lda : A + gi + gk * lda) : A, ok ? 8 : 0);
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int e = r * GT + tid;
      int j, kk;
      if (!TB) {
        kk = e % BK;
        j = e / BK;
      } else {
        j = e % TBN;
        kk = e / TBN;
      }
      const int64_t gj = tn + j, gk = k0 + kk;
      const bool ok = gj < n && gk < ke;
      gm_cp8(Bs + kk * LB + j, ok ? (TB ? B + gj + gk * ldb : B + gk + gj * ldb) : B, ok ? 8 : 0);
    }
  };

#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nk) issue(s);
    gm_commit();
  }
  for (int64_t t = 0; t < nk; ++t) {
    gm_wait<NSTAGE - 2>();  // k-tile t has landed (this thread's copies) ...
    __syncthreads();        // ... everyone's, and slot (t-1) % NSTAGE is free
    if (t + NSTAGE - 1 < nk) issue(t + NSTAGE - 1);
    gm_commit();
    const int slot = (int)(t % NSTAGE);
    const double *As = As0 + (size_t)slot * BK * LA;
    const double *Bs = Bs0 + (size_t)slot * BK * LB;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double a[MI], b[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = As[(ks + (lane & 3)) * LA + wm + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[j] = Bs[(ks + (lane & 3)) * LB + wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  gm_wait<0>();
  // epilogue
  double ss = 0.0;
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    int64_t row = tm + wm + i * 8 + (lane >> 2);
    if (row >= m) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int64_t col = tn + wn + j * 8 + 2 * (lane & 3) + h;
        if (col >= n) continue;
        if (EPI == 1) {
          const double r0 = c_trans ? C[col + row * ldc] : C[row + col * ldc];
          const double v = r0 - acc[i][j][h];
          ss += v * v;
        } else if (partial) {
          partial[((int64_t)blockIdx.z * n + col) * m + row] = acc[i][j][h];
        } else {
          double v = alpha * acc[i][j][h];
          if (beta != 0.0) v += beta * C[row + col * ldc];
          C[row + col * ldc] = v;
        }
      }
    }
  }
  // fused split-K reduction (tile_cnt != nullptr): the last of the tile's
  // gridDim.z CTAs to finish sums the partials in split order (fixed
  // association, so bit-reproducible) and resets the tile's counter
  if (EPI == 0 && partial && tile_cnt) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const unsigned tix = blockIdx.x + blockIdx.y * gridDim.x;
      const unsigned t = atomicAdd(tile_cnt + tix, 1u);
      s_last = t == gridDim.z - 1;
      if (s_last) tile_cnt[tix] = 0u;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      const int rows = (int)min((int64_t)TBM, m - tm), cols = (int)min((int64_t)TBN, n - tn);
      const int Z = (int)gridDim.z;
      for (int e = tid; e < rows * cols; e += GT) {
        const int c = e / rows, r = e - c * rows;
        const int64_t row = tm + r, col = tn + c;
        const double *pp = partial + col * m + row;
        const int64_t zs = n * m;
        double sacc = 0.0;
        int z = 0;
        for (; z + 8 <= Z; z += 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = __ldcg(pp + (int64_t)(z + u) * zs);
#pragma unroll
          for (int u = 0; u < 8; ++u) sacc += v[u];
        }
        for (; z < Z; ++z) sacc += __ldcg(pp + (int64_t)z * zs);
        double v = alpha * sacc;
        if (beta != 0.0) v += beta * C[row + col * ldc];
        C[row + col * ldc] = v;
      }
    }
  }
  if (EPI == 1) {
    __shared__ double s_ss[GT / 32];
#pragma unroll
    for (int off = 16; off; off >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, off);
    if (lane == 0) s_ss[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < GT / 32; ++w) t += s_ss[w];
      npart[blockIdx.x + (int64_t)blockIdx.y * gridDim.x] = t;
    }
    if (sum_out) last_cta_sum(npart, (int64_t)gridDim.x * gridDim.y, sum_out, tile_cnt);
  }
}

// ||R0 - Q B||_F^2 partials for a short inner dimension (k <= 64): a CTA
// owns 128 rows, keeps its Q rows in shared memory for the whole sweep over
// the column tiles (64 columns each, B tile staged per step), forms Q B on
// the DMMA pipe and reads every R0 element exactly once (RT: R0 stored
// transposed, R0(row, col) at R0[col + row * ldr]).  The general GEMM
// epilogue path re-read the Q tile for every 64x64 output tile, i.e.
// ~65x for the 314,928 x 4,160 operand of config 5.
template <bool RT>
__global__ void __launch_bounds__(128) k_resid_rows(int64_t m, int64_t n, int k, int kp,
                                                    const double *__restrict__ Q, int64_t ldq,
                                                    const double *__restrict__ B, int64_t ldb,
                                                    const double *__restrict__ R0, int64_t ldr,
                                                    int64_t tiles_per_cta,
                                                    double *__restrict__ npart,
                                                    double *__restrict__ sum_out,
                                                    unsigned *__restrict__ counter) {
  extern __shared__ double rs_smem[];
  double(*Qs)[128 + PAD] = reinterpret_cast<double(*)[128 + PAD]>(rs_smem);       // [kp][128]
  double(*Bs)[64 + PAD] = reinterpret_cast<double(*)[64 + PAD]>(rs_smem + (size_t)kp * (128 + PAD));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tm = (int64_t)blockIdx.x * 128;
  for (int e = tid; e < kp * 128; e += 128) {
    const int i = e % 128, kk = e / 128;
    const int64_t gi = tm + i;
    Qs[kk][i] = (gi < m && kk < k) ? Q[gi + (int64_t)kk * ldq] : 0.0;
  }
  double ss = 0.0;
  const int64_t t0 = (int64_t)blockIdx.y * tiles_per_cta;
  const int64_t t1 = min(ceil_div_dev(n, 64), t0 + tiles_per_cta);
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t tn = t * 64;
    __syncthreads();  // previous tile's Bs reads are done (and Qs is ready)
    for (int e = tid; e < kp * 64; e += 128) {
      const int kk = e % kp, j = e / kp;
      const int64_t gj = tn + j;
      Bs[kk][j] = (gj < n && kk < k) ? B[kk + gj * ldb] : 0.0;
    }
    __syncthreads();
    double acc[4][8][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int ks = 0; ks < kp; ks += 4) {
      double a[4], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Qs[ks + (lane & 3)][warp * 32 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[ks + (lane & 3)][j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t row = tm + warp * 32 + i * 8 + (lane >> 2);
      if (row >= m) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t col = tn + j * 8 + 2 * (lane & 3) + h;
          if (col >= n) continue;
          const double r0 = RT ? R0[col + row * ldr] : R0[row + col * ldr];
          const double v = r0 - acc[i][j][h];
          ss += v * v;
        }
    }
  }
  __shared__ double s_ss[4];
#pragma unroll
  for (int off = 16; off; off >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, off);
  if (lane == 0) s_ss[warp] = ss;
  __syncthreads();
  if (tid == 0) npart[blockIdx.x + (int64_t)blockIdx.y * gridDim.x] = (s_ss[0] + s_ss[1]) + (s_ss[2] + s_ss[3]);
  last_cta_sum(npart, (int64_t)gridDim.x * gridDim.y, sum_out, counter);
}

// Column-block variant for a column-major R0 (rows contiguous): a CTA owns
// 64 columns and a chunk of `rows_per_cta` rows, keeps its B tile in shared
// memory and steps down the rows 128 at a time (Q rows staged per step from
// L2), so every CTA streams 64 contiguous column segments -- the row-block
// order touched a new 2 MB page per 1 KB read on the 10.5 GB operand.
__global__ void __launch_bounds__(128) k_resid_cols(int64_t m, int64_t n, int k, int kp,
                                                    const double *__restrict__ Q, int64_t ldq,
                                                    const double *__restrict__ B, int64_t ldb,
                                                    const double *__restrict__ R0, int64_t ldr,
                                                    int64_t rows_per_cta,
                                                    double *__restrict__ npart,
                                                    double *__restrict__ sum_out,
                                                    unsigned *__restrict__ counter) {
  extern __shared__ double rs_smem[];
  double(*Qs)[128 + PAD] = reinterpret_cast<double(*)[128 + PAD]>(rs_smem);       // [kp][128]
  double(*Bs)[64 + PAD] = reinterpret_cast<double(*)[64 + PAD]>(rs_smem + (size_t)kp * (128 + PAD));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tn = (int64_t)blockIdx.x * 64;
  for (int e = tid; e < kp * 64; e += 128) {
    const int kk = e % kp, j = e / kp;
    const int64_t gj = tn + j;
    Bs[kk][j] = (gj < n && kk < k) ? B[kk + gj * ldb] : 0.0;
  }
  double ss = 0.0;
  const int64_t r_begin = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t r_end = min(m, r_begin + rows_per_cta);
  for (int64_t tm = r_begin; tm < r_end; tm += 128) {
    __syncthreads();
    for (int e = tid; e < kp * 128; e += 128) {
      const int i = e % 128, kk = e / 128;
      const int64_t gi = tm + i;
      Qs[kk][i] = (gi < r_end && kk < k) ? Q[gi + (int64_t)kk * ldq] : 0.0;
    }
    __syncthreads();
    double acc[4][8][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int ks = 0; ks < kp; ks += 4) {
      double a[4], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Qs[ks + (lane & 3)][warp * 32 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[ks + (lane & 3)][j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t row = tm + warp * 32 + i * 8 + (lane >> 2);
      if (row >= r_end) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t col = tn + j * 8 + 2 * (lane & 3) + h;
          if (col >= n) continue;
          const double v = R0[row + col * ldr] - acc[i][j][h];
          ss += v * v;
        }
    }
  }
  __shared__ double s_ss[4];
#pragma unroll
  for (int off = 16; off; off >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, off);
  if (lane == 0) s_ss[warp] = ss;
  __syncthreads();
  if (tid == 0) npart[blockIdx.x + (int64_t)blockIdx.y * gridDim.x] = (s_ss[0] + s_ss[1]) + (s_ss[2] + s_ss[3]);
  last_cta_sum(npart, (int64_t)gridDim.x * gridDim.y, sum_out, counter);
}

// Tile shape for an m x n output: the DMMA work of a tile is TBM x TBN
// whatever the valid part, so narrow outputs (a 40-wide sketch, a 16-rank
// core) get a tile whose short side just covers them -- a 64x64 tile spent
// 37% of config 5's largest product (104,976 x 40 x 512) on padding.
enum TileShape {
  T64x64 = 0, T128x32, T32x128, T128x16, T16x128, T128x40, T128x48, T48x128, T48x48, T32x32, T16x16
};
inline TileShape pick_tile(int64_t m, int64_t n) {
  if (m > 48 && n <= 48) {
    if (n <= 16) return T128x16;
    if (n <= 32) return T128x32;
    return n <= 40 ? T128x40 : T128x48;
  }
  if (n > 48 && m <= 48) return m <= 16 ? T16x128 : (m <= 32 ? T32x128 : T48x128);
  if (m <= 48 && n <= 48 && (m > 32 || n > 32)) return T48x48;
  if (m <= 32 && n <= 32) return m <= 16 && n <= 16 ? T16x16 : T32x32;
  return T64x64;
}
inline int tile_m(TileShape t) {
  switch (t) {
    case T128x32: case T128x16: case T128x40: case T128x48: return 128;
    case T32x128: return 32;
    case T16x128: return 16;
    case T48x128: case T48x48: return 48;
    case T32x32: return 32;
    case T16x16: return 16;
    default: return 64;
  }
}
inline int tile_n(TileShape t) {
  switch (t) {
    case T32x128: case T16x128: case T48x128: return 128;
    case T128x32: return 32;
    case T128x16: return 16;
    case T128x40: return 40;
    case T128x48: case T48x48: return 48;
    case T32x32: return 32;
    case T16x16: return 16;
    default: return 64;
  }
}

// one k_dgemm instantiation: opt in to its dynamic shared memory once
template <bool TA, bool TB, int EPI, int TBM, int TBN, typename... Args>
void launch_dgemm(dim3 grid, cudaStream_t st, Args... args) {
  constexpr size_t smem = gemm_smem_bytes(TBM, TBN);
  static const cudaError_t attr = cudaFuncSetAttribute(
      k_dgemm<TA, TB, EPI, TBM, TBN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  (void)attr;
  k_dgemm<TA, TB, EPI, TBM, TBN><<<grid, GT, smem, st>>>(args...);
}

// Deterministic split-K reduction.  Block = 64 outputs x G split groups
// (G = blockDim / 64: 4, or 16 for > 256 splits): thread (o, g) sums the
// contiguous group g of the partials of output o in split order (loads
// unrolled 8 deep so they are in flight together), then the G group sums
// are added in group order.  G is a function of `splits`, so the
// association is fixed and results are bit-reproducible.
constexpr int SR_OUT = 64, SR_GRP_MAX = 16;
inline int splitk_reduce_threads(int splits) { return SR_OUT * (splits > 256 ? 16 : 4); }
__global__ void __launch_bounds__(SR_OUT *SR_GRP_MAX) k_splitk_reduce(
    int64_t m, int64_t n, int splits, const double *__restrict__ partial, double alpha, double beta,
    double *__restrict__ C, int64_t ldc) {
  __shared__ double gs[SR_GRP_MAX][SR_OUT];
  const int64_t total = m * n;
  const int SR_GRP = (int)blockDim.x / SR_OUT;
  const int o = threadIdx.x % SR_OUT, g = threadIdx.x / SR_OUT;
  const int per = (splits + SR_GRP - 1) / SR_GRP;
  const int z0 = g * per, z1 = min(splits, z0 + per);
  for (int64_t base = (int64_t)blockIdx.x * SR_OUT; base < total; base += (int64_t)gridDim.x * SR_OUT) {
    const int64_t t = base + o;
    double s = 0.0;
    if (t < total) {
      int z = z0;
      for (; z + 8 <= z1; z += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(partial + (int64_t)(z + u) * total + t);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
      }
      for (; z < z1; ++z) s += __ldcg(partial + (int64_t)z * total + t);
    }
    gs[g][o] = s;
    __syncthreads();
    if (g == 0 && t < total) {
      double tot = gs[0][o];
      for (int q = 1; q < SR_GRP; ++q) tot += gs[q][o];
      const int64_t col = t / m, row = t - col * m;
      double v = alpha * tot;
      if (beta != 0.0) v += beta * C[row + col * ldc];
      C[row + col * ldc] = v;
    }
    __syncthreads();
  }
}

__global__ void k_scale_c(int64_t m, int64_t n, double beta, double *C, int64_t ldc) {
  int64_t total = m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t col = t / m, row = t - col * m;
    C[row + col * ldc] = beta == 0.0 ? 0.0 : beta * C[row + col * ldc];
  }
}

__global__ void k_transpose(int64_t rows, int64_t cols, const double *__restrict__ src, int64_t lds,
                            double *__restrict__ dst, int64_t ldd) {
  __shared__ double t[32][33];
  int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    int64_t r = r0 + threadIdx.x, c = c0 + j;
    if (r < rows && c < cols) t[j][threadIdx.x] = src[r + c * lds];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    int64_t c = c0 + threadIdx.x, r = r0 + j;  // dst(c, r) = src(r, c)
    if (r < rows && c < cols) dst[c + r * ldd] = t[threadIdx.x][j];
  }
}

__global__ void k_orth_defect(int64_t n, const double *__restrict__ G, int64_t ldg,
                              double *__restrict__ partial) {
  double mx = 0.0;
  int64_t total = n * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / n, i = t - j * n;
    double v = fabs(G[i + j * ldg] - (i == j ? 1.0 : 0.0));
    mx = fmax(mx, v);
  }
  for (int off = 16; off; off >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, off));
  __shared__ double s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, s[w]);
    partial[blockIdx.x] = t;
  }
}

}  // namespace

// K splits for a product with `tiles` output tiles: long-K products with a
// small output (Gram matrices, B = Q^T A, train-norm contractions) otherwise
// run a handful of CTAs that walk all of K one BK step at a time (latency
// bound, ~0.7 us per step).  Aim for ~8 CTAs per SM, at least 128 K per CTA
// (8 BK steps), at most 256 splits (the reduction's serial depth) -- 1024
// for tiles of <= 1024 outputs, whose per-split DMMA work is small (the
// 32 x 32 Gram of a 314,928-row panel ran 77 k-steps per CTA at 256).
int64_t splitk_count(int64_t tiles, int64_t k, int num_sms, int64_t tile_elems) {
  if (tiles >= 2 * (int64_t)num_sms || k < 512) return 1;
  int64_t s = ceil_div(8 * (int64_t)num_sms, tiles);
  s = std::min<int64_t>(s, k / 128);
  s = std::min<int64_t>(s, tile_elems <= 1024 ? 1024 : (tile_elems <= 2048 ? 512 : 256));
  return std::max<int64_t>(s, 1);
}

int gemm(ftt_ctx *ctx, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha,
         const double *A, int64_t lda, const double *B, int64_t ldb, double beta, double *C,
         int64_t ldc, double *splitk_ws, size_t splitk_ws_elems) {
  if (m <= 0 || n <= 0) return FTT_OK;
  if (k <= 0 || alpha == 0.0) {
    if (beta == 1.0) return FTT_OK;
    k_scale_c<<<grid_for(m * n, 256, 4), 256, 0, ctx->stream>>>(m, n, beta, C, ldc);
    FTT_LAUNCHED(ctx);
    return FTT_OK;
  }
  const TileShape ts = pick_tile(m, n);
  int64_t tiles_m = ceil_div(m, tile_m(ts)), tiles_n = ceil_div(n, tile_n(ts));
  int64_t tiles = tiles_m * tiles_n;
  int splits = 1;
  {
    int64_t s = splitk_count(tiles, k, ctx->num_sms, (int64_t)tile_m(ts) * tile_n(ts));
    if (splitk_ws) s = std::min<int64_t>(s, (int64_t)(splitk_ws_elems / (size_t)(m * n)));
    else s = 1;
    if (s > 1) splits = (int)s;
  }
  int64_t kps = ceil_div(ceil_div(k, splits), BK) * BK;
  splits = (int)ceil_div(k, kps);
  if (tiles_m > 65535 * 1024LL || tiles_n > 65535) {
    set_error("gemm: grid too large (%lld x %lld tiles)", (long long)tiles_m, (long long)tiles_n);
    return FTT_ERR_INVALID;
  }
  dim3 grid((unsigned)tiles_m, (unsigned)tiles_n, (unsigned)splits);
  double *part = splits > 1 ? splitk_ws : nullptr;
  // small outputs: the last CTA per tile reduces (no second launch); the
  // serial depth stays <= ~256 loads per thread of that CTA
  const int64_t tile_elems = std::min<int64_t>(m, tile_m(ts)) * std::min<int64_t>(n, tile_n(ts));
  static const bool no_fuse = getenv("FTT_NO_SPLITK_FUSE") != nullptr;
  unsigned *tcnt = (splits > 1 && !no_fuse && ctx->tile_cnt && tiles <= kTileCnt &&
                    tile_elems * splits <= 256 * GT)
                       ? ctx->tile_cnt
                       : nullptr;
  static const bool dbg = getenv("FTT_DEBUG_GEMM") != nullptr;
  cudaEvent_t dev[2];
  if (dbg) {
    cudaEventCreate(&dev[0]);
    cudaEventCreate(&dev[1]);
    cudaEventRecord(dev[0], ctx->stream);
  }
  const int pb = prof_begin(ctx);
#define FTT_GEMM_LAUNCH(TA_, TB_, M_, N_)                                                     \
  launch_dgemm<TA_, TB_, 0, M_, N_>(grid, ctx->stream, m, n, k, alpha, A, lda, B, ldb, beta, C, \
                                    ldc, kps, part, 0, (double *)nullptr, tcnt, (double *)nullptr)
#define FTT_GEMM_TILES(TA_, TB_)                                         \
  do {                                                                   \
    switch (ts) {                                                        \
      case T128x32: FTT_GEMM_LAUNCH(TA_, TB_, 128, 32); break;           \
      case T32x128: FTT_GEMM_LAUNCH(TA_, TB_, 32, 128); break;           \
      case T128x16: FTT_GEMM_LAUNCH(TA_, TB_, 128, 16); break;           \
      case T16x128: FTT_GEMM_LAUNCH(TA_, TB_, 16, 128); break;           \
      case T128x40: FTT_GEMM_LAUNCH(TA_, TB_, 128, 40); break;           \
      case T128x48: FTT_GEMM_LAUNCH(TA_, TB_, 128, 48); break;           \
      case T48x128: FTT_GEMM_LAUNCH(TA_, TB_, 48, 128); break;           \
      case T48x48: FTT_GEMM_LAUNCH(TA_, TB_, 48, 48); break;             \
      case T32x32: FTT_GEMM_LAUNCH(TA_, TB_, 32, 32); break;             \
      case T16x16: FTT_GEMM_LAUNCH(TA_, TB_, 16, 16); break;             \
      default: FTT_GEMM_LAUNCH(TA_, TB_, 64, 64); break;                 \
    }                                                                    \
  } while (0)
  if (!ta && !tb) FTT_GEMM_TILES(false, false);
  else if (!ta && tb) FTT_GEMM_TILES(false, true);
  else if (ta && !tb) FTT_GEMM_TILES(true, false);
  else FTT_GEMM_TILES(true, true);
#undef FTT_GEMM_TILES
#undef FTT_GEMM_LAUNCH
  FTT_LAUNCHED(ctx);
  if (splits > 1 && !tcnt) {
    const int64_t rb = std::min<int64_t>(ceil_div(m * n, SR_OUT), 4 * (int64_t)ctx->num_sms);
    k_splitk_reduce<<<(unsigned)rb, splitk_reduce_threads(splits), 0, ctx->stream>>>(
        m, n, splits, part, alpha, beta, C, ldc);
    FTT_LAUNCHED(ctx);
  }
  prof_end(ctx, pb, PT_GEMM, 8.0 * ((double)m * k + (double)k * n + 2.0 * m * n),
           2.0 * (double)m * n * k);
  if (dbg) {
    cudaEventRecord(dev[1], ctx->stream);
    cudaEventSynchronize(dev[1]);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, dev[0], dev[1]);
    fprintf(stderr, "[gemm] %c%c m=%lld n=%lld k=%lld tile=%d splits=%d %.1f us %.2f TF/s\n",
            ta ? 'T' : 'N', tb ? 'T' : 'N', (long long)m, (long long)n, (long long)k, (int)ts,
            splits, 1e3 * ms, 2.0 * m * n * k / (ms * 1e-3) / 1e12);
    cudaEventDestroy(dev[0]);
    cudaEventDestroy(dev[1]);
  }
  return FTT_OK;
}

namespace {
__global__ void __launch_bounds__(256) k_dmma_peak(int64_t iters, double seed, double *out) {
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  double a = seed * (1 + (threadIdx.x & 7)), b = seed * (1 + (threadIdx.x >> 5));
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(acc[j][0], acc[j][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1];
  if (s == 1234.5678) out[0] = s;  // keep the chain alive
}
}  // namespace

int bench_dmma(ftt_ctx *ctx, int64_t iters, double *tflops) {
  FTT_CHECK(arena_reserve(ctx, 256));
  double *sink = take<double>(ctx, 1);
  cudaEvent_t e0, e1;
  FTT_CUDA(cudaEventCreate(&e0));
  FTT_CUDA(cudaEventCreate(&e1));
  const int blocks = ctx->num_sms * 4;
  k_dmma_peak<<<blocks, 256, 0, ctx->stream>>>(iters / 10 + 1, 1e-3, sink);  // warm-up
  FTT_LAUNCHED(ctx);
  FTT_CUDA(cudaEventRecord(e0, ctx->stream));
  k_dmma_peak<<<blocks, 256, 0, ctx->stream>>>(iters, 1e-3, sink);
  FTT_LAUNCHED(ctx);
  FTT_CUDA(cudaEventRecord(e1, ctx->stream));
  FTT_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  FTT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  // 8 warps x 8 chains x iters DMMAs, 512 flops each
  double flops = (double)blocks * 8 * 8 * (double)iters * 512.0;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return FTT_OK;
}

// ||R0 - op(A) op(B)||_F^2 (m x n, inner k) without writing the residual;
// deterministic (fixed tile grid, fixed-order reduction).
int gemm_resid_sumsq(ftt_ctx *ctx, int ta, int tb, int64_t m, int64_t n, int64_t k,
                     const double *A, int64_t lda, const double *B, int64_t ldb, const double *R0,
                     int64_t ldr, int r_trans, double *out_host, double *out_dev) {
  if (out_host) *out_host = 0.0;
  if (m <= 0 || n <= 0) {
    if (out_dev) FTT_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double), ctx->stream));
    return FTT_OK;
  }
  if (!ta && !tb && k >= 1 && k <= 64) {
    // short inner dimension: Q / B tiles resident in shared memory, R0 read
    // once in its contiguous direction (rows for a transposed R0, columns
    // otherwise)
    const int kp = (int)ceil_div(k, 4) * 4;
    static bool attr = false;
    if (!attr) {
      const int mx = 8 * 64 * (128 + PAD + 64 + PAD);
      FTT_CUDA(cudaFuncSetAttribute(k_resid_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
      FTT_CUDA(cudaFuncSetAttribute(k_resid_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
      attr = true;
    }
    const size_t smem = 8 * (size_t)kp * (128 + PAD + 64 + PAD);
    dim3 grid;
    int64_t per = 0;
    if (r_trans) {
      const int64_t rb = ceil_div(m, 128), ct = ceil_div(n, 64);
      const int64_t chunks = std::min<int64_t>(ct, std::max<int64_t>(1, ceil_div(4 * ctx->num_sms, rb)));
      per = ceil_div(ct, chunks);
      grid = dim3((unsigned)rb, (unsigned)ceil_div(ct, per));
    } else {
      const int64_t cb = ceil_div(n, 64);
      // row chunks: >= 8 CTAs per SM overall, >= 128 rows each
      const int64_t want = std::max<int64_t>(1, ceil_div(8 * ctx->num_sms, cb));
      per = std::max<int64_t>(128, ceil_div(ceil_div(m, want), 128) * 128);
      grid = dim3((unsigned)cb, (unsigned)ceil_div(m, per));
    }
    const int64_t nt = (int64_t)grid.x * grid.y;
    double *npart = nullptr;
    FTT_CHECK(owned_alloc(ctx, (void **)&npart, 8 * (size_t)(nt + 1)));
    const int pb = prof_begin(ctx);
    double *sum = out_dev ? out_dev : npart + nt;
    unsigned *cnt = ctx->tile_cnt + kTileCnt + 1;
    if (r_trans)
      k_resid_rows<true><<<grid, 128, smem, ctx->stream>>>(m, n, (int)k, kp, A, lda, B, ldb, R0, ldr,
                                                           per, npart, sum, cnt);
    else
      k_resid_cols<<<grid, 128, smem, ctx->stream>>>(m, n, (int)k, kp, A, lda, B, ldb, R0, ldr, per,
                                                     npart, sum, cnt);
    FTT_LAUNCHED(ctx);
    prof_end(ctx, pb, PT_GEMM, 8.0 * ((double)m * n + (double)m * k + (double)k * n),
             2.0 * (double)m * n * k);
    if (out_host) FTT_CHECK(copy_to_host(ctx, out_host, npart + nt, sizeof(double)));
    owned_free(ctx, npart);
    return FTT_OK;
  }
  const int64_t tiles_m = ceil_div(m, BM), tiles_n = ceil_div(n, BN);
  if (tiles_n > 65535) {
    set_error("gemm_resid_sumsq: too many column tiles");
    return FTT_ERR_INVALID;
  }
  const int64_t nt = tiles_m * tiles_n;
  double *npart = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&npart, 8 * (size_t)(nt + 1)));
  dim3 grid((unsigned)tiles_m, (unsigned)tiles_n, 1);
  const int64_t kps = ceil_div(std::max<int64_t>(k, 1), BK) * BK;
  double *C = const_cast<double *>(R0);
  double *sum = out_dev ? out_dev : npart + nt;
  unsigned *cnt = ctx->tile_cnt + kTileCnt + 1;
#define FTT_RESID_LAUNCH(TA_, TB_)                                                              \
  launch_dgemm<TA_, TB_, 1, 64, 64>(grid, ctx->stream, m, n, k, 1.0, A, lda, B, ldb, 0.0, C, ldr, \
                                    kps, (double *)nullptr, r_trans, npart, cnt, sum)
  if (!ta && !tb) FTT_RESID_LAUNCH(false, false);
  else if (!ta && tb) FTT_RESID_LAUNCH(false, true);
  else if (ta && !tb) FTT_RESID_LAUNCH(true, false);
  else FTT_RESID_LAUNCH(true, true);
#undef FTT_RESID_LAUNCH
  FTT_LAUNCHED(ctx);
  if (out_host) FTT_CHECK(copy_to_host(ctx, out_host, npart + nt, sizeof(double)));
  owned_free(ctx, npart);
  return FTT_OK;
}

size_t gemm_splitk_elems(int64_t m, int64_t n, int64_t k) {
  const TileShape ts = pick_tile(m, n);
  int64_t tiles = ceil_div(m, tile_m(ts)) * ceil_div(n, tile_n(ts));
  int64_t s = splitk_count(tiles, k, kNumSMs, (int64_t)tile_m(ts) * tile_n(ts));
  return s > 1 ? (size_t)(s * m * n) : 0;
}

int transpose(ftt_ctx *ctx, int64_t rows, int64_t cols, const double *src, int64_t lds, double *dst,
              int64_t ldd) {
  if (rows <= 0 || cols <= 0) return FTT_OK;
  dim3 grid((unsigned)ceil_div(rows, 32), (unsigned)ceil_div(cols, 32));
  k_transpose<<<grid, dim3(32, 8), 0, ctx->stream>>>(rows, cols, src, lds, dst, ldd);
  FTT_LAUNCHED(ctx);
  return FTT_OK;
}

}  // namespace ftt

using namespace ftt;

extern "C" {

int ftt_dgemm(ftt_ctx *ctx, int32_t transa, int32_t transb, int64_t m, int64_t n, int64_t k,
              double alpha, const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
              double *C, int64_t ldc) {
  if (!ctx || m < 0 || n < 0 || k < 0) {
    set_error("ftt_dgemm: invalid sizes");
    return FTT_ERR_INVALID;
  }
  size_t ws = gemm_splitk_elems(m, n, k);
  double *part = nullptr;
  if (ws) {
    FTT_CHECK(arena_reserve(ctx, align_up(ws * sizeof(double))));
    part = take<double>(ctx, ws);
  }
  return gemm(ctx, transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, part, ws);
}

int ftt_bench_dmma(ftt_ctx *ctx, int64_t iters, double *tflops_out) {
  if (!ctx || !tflops_out || iters < 1) return FTT_ERR_INVALID;
  return bench_dmma(ctx, iters, tflops_out);
}

int ftt_orth_defect(ftt_ctx *ctx, int64_t n, const double *G, int64_t ldg, double *out_host) {
  if (!ctx || !out_host || n < 0) return FTT_ERR_INVALID;
  *out_host = 0.0;
  if (n == 0) return FTT_OK;
  int nb = grid_for(n * n, 256, 4, 1024);
  FTT_CHECK(arena_reserve(ctx, align_up(8 * nb) + 256));
  double *part = take<double>(ctx, nb);
  k_orth_defect<<<nb, 256, 0, ctx->stream>>>(n, G, ldg, part);
  FTT_LAUNCHED(ctx);
  std::vector<double> h(nb);
  FTT_CHECK(copy_to_host(ctx, h.data(), part, 8 * nb));
  double mx = 0.0;
  for (double v : h) mx = v > mx ? v : mx;
  *out_host = mx;
  return FTT_OK;
}

int ftt_transpose(ftt_ctx *ctx, int64_t rows, int64_t cols, const double *src, int64_t lds,
                  double *dst, int64_t ldd) {
  if (!ctx) return FTT_ERR_INVALID;
  return transpose(ctx, rows, cols, src, lds, dst, ldd);
}

}  // extern "C"
