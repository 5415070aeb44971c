// Narrow dense fp64 factorisations (n <= 64 columns) without grid-wide
// synchronisation: the latency path of the rounding sweeps.
//
// The truncation SVDs of the BASELINE configs are mostly tall and narrow
// (512 x 24, 10366 x 24 sketches, 62206 x 32, 314928 x 32, 4160 x 32 ...).
// A blocked Householder QR with a cooperative panel pays a grid barrier per
// column; here every step stays inside one CTA and the matrix stays in
// REGISTERS, one row per thread:
//
//   reg_qr      Householder QR with a rotating row layout (the active column
//               is always register 0; the row shifts left after each step,
//               so indices are static and the loop body is one compact code
//               block).  Per column: each thread forms its row's contribution
//               to |x|^2 and to the dots with the trailing columns, a warp
//               reduce-scatter (lane j <- warp sum of slot j) and a shared
//               array of per-warp partials give the totals after one
//               barrier; the threads j in [c, n) compute tau / beta and
//               w_j = tau (a_cj + v^T a_j) in a FIXED warp order (bit-identical
//               scalars everywhere, deterministic), a second barrier
//               publishes them, every thread updates its own row.
//   apply_q     Z <- Q Z for a Z held row-wise in registers, reflectors read
//               from shared memory (Q_thin = Q [I; 0]), same two-barrier step.
//   cta_jacobi  one-sided (Hestenes) Jacobi on an n x n block in shared
//               memory, round-robin pairs, a warp per pair, fresh dots for
//               every rotation, one barrier per round.
//   TSQR        a tall matrix is cut into row blocks of 256 (one CTA each):
//               A_b = Q_b R_b, the stacked R_b are reduced the same way
//               until one block remains; Q (or U = Q P) is expanded back
//               down the tree with small batched products.
//
// SVD of a narrow A_tall = Q R (TSQR, root R sign-fixed): X = R^T, X P = Y
// (k_jacobi_small), sigma_j = ||Y_j||, U_A = Q P (Q_root P expanded down the
// tree), V_A = Y / sigma (as in ftt_svd.cu).
#include <algorithm>
#include <vector>

#include "ftt_dense.cuh"
#include "ftt_small.cuh"

namespace ftt {
namespace {

constexpr double kEps = 2.220446049250313e-16;
constexpr int LEAF_NT = 256;  // TSQR / QR kernels: 256 threads, one row each ...
constexpr int LEAF_MAX = 512; // ... 512 for n <= 16 (half the leaves, fewer tree levels)
inline int leaf_rows(int n) { return n <= 16 ? LEAF_MAX : LEAF_NT; }
constexpr int SVD_NT = 1024;  // SVD kernel: 32 warps, one per pair of a Jacobi round (n <= 64)

__device__ __forceinline__ double warp_sum(double v) {
  // butterfly: every lane ends with the bit-identical total (fp add commutes)
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// W per-lane slots (W = 8, 16, 32) -> lane l receives the warp-wide sum of
// slot l mod W: lanes differing in the bits >= log2(W) are folded first,
// then a halving exchange (at offset s each lane keeps the upper or lower s
// slots by bit s of its lane id and adds the partner's copy).
template <int W>
__device__ __forceinline__ double reduce_scatter(double (&v)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= W; o >>= 1)
#pragma unroll
    for (int j = 0; j < W; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
#pragma unroll
  for (int s = W / 2; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int j = 0; j < s; ++j) {
      const double send = upper ? v[j] : v[j + s];
      const double keep = upper ? v[j + s] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

template <int NMAX>
struct Scratch {
  double red[LEAF_MAX / 32][NMAX];  // per-warp partial sums (QR kernels: <= LEAF_MAX threads)
  double rowc[NMAX];              // row c (pivot row) of the current step
  double wv[NMAX];                // w_j of the current step
  double sc[4];                   // tau, beta, scal
  double tau[NMAX];
  double beta[NMAX];              // diagonal of R
};

// Column sums over the CTA of x * b[t] (t < NMAX) -> red[warp][t], in chunks
// of up to 32 slots (warp reduce-scatter: lane l ends with the warp sum of
// slot l).
template <int NMAX, int H, int W>
__device__ __forceinline__ void chunk_partials(double (*red)[NMAX], double x, const double (&b)[NMAX],
                                               int lane, int warp) {
  double p[32];
#pragma unroll
  for (int t = 0; t < 32; ++t) p[t] = (t < W && H + t < NMAX) ? x * b[H + t] : 0.0;
  const double tot = reduce_scatter<W>(p, lane);
  if (lane < W && H + lane < NMAX) red[warp][H + lane] = tot;
}

template <int NMAX>
__device__ __forceinline__ void block_partials(double (*red)[NMAX], double x,
                                               const double (&b)[NMAX]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int W0 = NMAX >= 24 ? 32 : (NMAX > 8 ? 16 : 8);
  chunk_partials<NMAX, 0, W0>(red, x, b, lane, warp);
  if constexpr (NMAX > 32) chunk_partials<NMAX, 32, (NMAX - 32 > 16 ? 32 : 16)>(red, x, b, lane, warp);
}

template <int NMAX>
__device__ __forceinline__ double sum_warps(const double (*red)[NMAX], int j) {
  const int nw = blockDim.x >> 5;
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += red[w][j];
  return t;
}

// Householder QR of the m x n block held row-wise in registers, one row per
// thread (row i = threadIdx.x).  Rotating layout: at step c, a[t] holds
// column c + t of the row; once the step is done the finished column-c entry
// is stored to Sref(i, c) (ld m) and the row shifts left by one, so the loop
// body is the same code for every c.  (A fully unrolled variant with static
// column indices spent most of its cycles waiting on instruction fetch.)
// On exit Sref holds LAPACK's dgeqrf layout for columns < min(m, n) and
// a[t] column min(m, n) + t; sc.tau / sc.beta the taus and diag(R).
template <int NMAX>
__device__ void reg_qr(double (&a)[NMAX], int m, int n, double *Sref, Scratch<NMAX> &sc) {
  const int i = threadIdx.x;
  const int k = min(m, n);
  for (int c = 0; c < k; ++c) {
    const int nc = n - c;  // live columns t < nc
    if (i == c) {
#pragma unroll
      for (int t = 0; t < NMAX; ++t) sc.rowc[t] = a[t];
    }
    block_partials<NMAX>(sc.red, (i > c && i < m) ? a[0] : 0.0, a);
    __syncthreads();
    if (i < nc) {  // thread t: column c + t (t = 0: the pivot's scalars)
      const double xx = sum_warps<NMAX>(sc.red, 0);
      const double alpha = sc.rowc[0];
      double tau, beta, scal;
      if (xx == 0.0) {
        tau = 0.0;
        beta = alpha;
        scal = 0.0;
      } else {
        beta = -copysign(sqrt(alpha * alpha + xx), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      if (i == 0) {
        sc.tau[c] = tau;
        sc.beta[c] = beta;
        sc.sc[0] = tau;
        sc.sc[1] = beta;
        sc.sc[2] = scal;
      } else {
        sc.wv[i] = tau * (sc.rowc[i] + scal * sum_warps<NMAX>(sc.red, i));
      }
    }
    __syncthreads();
    const double tau = sc.sc[0], beta = sc.sc[1], scal = sc.sc[2];
    if (i > c && i < m) {
      const double v = scal * a[0];
      if (tau != 0.0) {
#pragma unroll
        for (int t = 1; t < NMAX; ++t)
          if (t < nc) a[t] -= sc.wv[t] * v;
      }
      a[0] = v;
    } else if (i == c) {
      if (tau != 0.0) {
#pragma unroll
        for (int t = 1; t < NMAX; ++t)
          if (t < nc) a[t] -= sc.wv[t];
      }
      a[0] = beta;
    }
    if (i < m) Sref[i + (size_t)c * m] = a[0];
#pragma unroll
    for (int t = 0; t + 1 < NMAX; ++t) a[t] = a[t + 1];
    a[NMAX - 1] = 0.0;
  }
  __syncthreads();
}

// z <- Q z for z (one row per thread in registers, columns < ncol) with the
// reflectors of a k-column factorisation in Sref (ld m): c = k-1 .. 0.
template <int NMAX>
__device__ void apply_q(const double *Sref, const double *tau_s, double (&z)[NMAX], int m, int k,
                        int ncol, Scratch<NMAX> &sc) {
  const int i = threadIdx.x;
  for (int c = k - 1; c >= 0; --c) {
    const double tau = tau_s[c];
    if (tau == 0.0) continue;
    const double v = i == c ? 1.0 : ((i > c && i < m) ? Sref[i + (size_t)c * m] : 0.0);
    block_partials<NMAX>(sc.red, v, z);
    __syncthreads();
    if (i < ncol) sc.wv[i] = tau * sum_warps<NMAX>(sc.red, i);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
      if (j < ncol) z[j] -= sc.wv[j] * v;
  }
  __syncthreads();
}

__device__ __forceinline__ void rr_pair(int ne, int round, int c, int *p, int *q) {
  // circle method over ne (even) players, player ne-1 fixed
  const int L = ne - 1;
  if (c == 0) {
    *p = round;
    *q = L;
  } else {  // (round + c) mod L and (round - c) mod L without integer division
    const int x = round + c, y = round - c;
    *p = x >= L ? x - L : x;
    *q = y < 0 ? y + L : y;
  }
}

// One-sided Jacobi on X (n x n, ld n) accumulating P (n x n, ld n), both in
// shared memory; a warp per pair.  Convergence rule as the block kernel
// (ftt_svd.cu): a pair rotates iff both columns are above the noise floor and
// |x_p . x_q| > tol sqrt(|x_p|^2 |x_q|^2).  The rotation is exact by
// construction (c = 1/sqrt(1 + t^2), s = c t), so t only steers convergence.
// Returns the sweeps used (-1 if max_sweeps was exhausted).
__device__ int cta_jacobi(double *X, double *P, int n, double tol, double floor, int max_sweeps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ne = n + (n & 1);
  const int npairs = ne / 2;
  __syncthreads();
  for (int sw = 0; sw < max_sweeps; ++sw) {
    int any = 0;
    for (int round = 0; round < ne - 1; ++round) {
      for (int pi = warp; pi < npairs; pi += nw) {
        int p, q;
        rr_pair(ne, round, pi, &p, &q);
        if (p >= n || q >= n) continue;
        double *xp = X + (size_t)p * n, *xq = X + (size_t)q * n;
        const double u0 = lane < n ? xp[lane] : 0.0, v0 = lane < n ? xq[lane] : 0.0;
        const bool two = lane + 32 < n;
        const double u1 = two ? xp[lane + 32] : 0.0, v1 = two ? xq[lane + 32] : 0.0;
        double a = u0 * u0 + u1 * u1, b = v0 * v0 + v1 * v1, g = u0 * v0 + u1 * v1;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        if (a > floor && b > floor && fabs(g) > tol * sqrt(a * b)) {
          const double zeta = (b - a) / (2.0 * g);
          const double t = copysign(1.0 / (fabs(zeta) + sqrt(1.0 + zeta * zeta)), zeta);
          const double c = rsqrt(1.0 + t * t);
          const double s = c * t;
          double *pp = P + (size_t)p * n, *pq = P + (size_t)q * n;
          if (lane < n) {
            xp[lane] = c * u0 - s * v0;
            xq[lane] = s * u0 + c * v0;
            const double pu = pp[lane], pv = pq[lane];
            pp[lane] = c * pu - s * pv;
            pq[lane] = s * pu + c * pv;
          }
          if (two) {
            xp[lane + 32] = c * u1 - s * v1;
            xq[lane + 32] = s * u1 + c * v1;
            const double pu = pp[lane + 32], pv = pq[lane + 32];
            pp[lane + 32] = c * pu - s * pv;
            pq[lane + 32] = s * pu + c * pv;
          }
          any = 1;
        }
      }
      if (round < ne - 2) __syncthreads();
    }
    if (!__syncthreads_or(any)) return sw + 1;
  }
  return -1;
}

// Block reduction with a fixed order (deterministic).
__device__ double cta_sum(double v, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  return t;
}

// Row r0 + threadIdx.x of A_tall into registers (zero past the block / past
// column n).  A_tall is `buf` column-major (ld) or its transpose (trans).
// Returns false (in every thread) on a non-finite entry.
template <int NMAX>
__device__ bool load_row(double (&a)[NMAX], int mb, int n, const double *__restrict__ buf, int64_t ld,
                         int trans, int64_t r0) {
  int bad = 0;
  const int i = threadIdx.x;
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    double v = 0.0;
    if (i < mb && j < n) v = trans ? buf[j + (r0 + i) * ld] : buf[(r0 + i) + (int64_t)j * ld];
    bad |= !isfinite(v);
    a[j] = v;
  }
  return !__syncthreads_or(bad);
}

// ---- kernels ----------------------------------------------------------

// TSQR level: CTA b factors rows [b L, min(M, (b+1) L)) (L = 256) of A_tall,
// writes R_b (n x n, zero below the diagonal and below row m_b) into rows
// [b n, (b+1) n) of Rs (ld ldr) and Q_b (m_b x n) into the same rows of Qo
// (ld ldq).  With `root`, R gets diag >= 0 (row signs folded into Q's
// columns) -- the sign convention of qr_economic.  Q_b = H_0 .. H_{k-1} [I; 0]
// is formed from the reflectors staged in shared memory (dynamic, m_b x n).
// status[0] |= 1 on a non-finite input.
template <int NMAX>
__global__ void __launch_bounds__(NMAX <= 16 ? LEAF_MAX : LEAF_NT, 1) k_tsqr_level(int64_t M, int n,
                                                            const double *__restrict__ A,
                                                            int64_t lda, int trans,
                                                            double *__restrict__ Rs, int64_t ldr,
                                                            double *__restrict__ Qo, int64_t ldq,
                                                            int root, int *__restrict__ status) {
  extern __shared__ double Sref[];
  __shared__ Scratch<NMAX> sc;
  const int64_t r0 = (int64_t)blockIdx.x * blockDim.x;  // leaf rows = threads (grid > 1)
  const int mb = (int)min((int64_t)blockDim.x, M - r0);
  const int k = min(mb, n);
  const int i = threadIdx.x;
  double a[NMAX];
  if (!load_row<NMAX>(a, mb, n, A, lda, trans, r0)) {
    if (i == 0) atomicOr(status, 1);
    return;
  }
  reg_qr<NMAX>(a, mb, n, Sref, sc);
  if (i < mb) {  // columns k.. (only when the block is wider than tall)
#pragma unroll
    for (int t = 0; t < NMAX; ++t)
      if (k + t < n) Sref[i + (size_t)(k + t) * mb] = a[t];
  }
  __syncthreads();
  if (Rs && i < n) {  // row i of R_b (sign-fixed at the root)
    const double sg = (root && i < k && sc.beta[i] < 0.0) ? -1.0 : 1.0;
    const int64_t rb = (int64_t)blockIdx.x * n + i;
    for (int j = 0; j < n; ++j)
      Rs[rb + (int64_t)j * ldr] = (i <= j && i < mb) ? sg * Sref[i + (size_t)j * mb] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < NMAX; ++j) a[j] = (i == j && j < k) ? 1.0 : 0.0;
  apply_q<NMAX>(Sref, sc.tau, a, mb, k, k, sc);
  if (i < mb) {
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
      if (j < n) {
        const double sg = (root && j < k && sc.beta[j] < 0.0) ? -1.0 : 1.0;
        Qo[(r0 + i) + (int64_t)j * ldq] = j < k ? sg * a[j] : 0.0;
      }
  }
}

// Jacobi stage of the narrow SVD: X = R^T (R n x n, ld ldr), X P = Y.
// Writes Y, P (n x n, ld n) and norms_j = ||Y_j||; status[0] |= 2 on no
// convergence, status[1] = sweeps.
__global__ void __launch_bounds__(SVD_NT) k_jacobi_small(int n, const double *__restrict__ R,
                                                         int64_t ldr, double *__restrict__ Yo,
                                                         double *__restrict__ Po,
                                                         double *__restrict__ norms,
                                                         int max_sweeps, int *__restrict__ status) {
  extern __shared__ double S[];  // X n x n | P n x n
  __shared__ double red[SVD_NT / 32];
  double *X = S;
  double *P = S + (size_t)n * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double f = 0.0;
  for (int e = tid; e < n * n; e += (int)blockDim.x) {
    const int j = e / n, i = e - j * n;  // X(i, j) = R(j, i)
    const double v = j <= i ? R[j + (int64_t)i * ldr] : 0.0;
    X[e] = v;
    P[e] = i == j ? 1.0 : 0.0;
    f += v * v;
  }
  const double fro2 = cta_sum(f, red);
  __syncthreads();
  const double tol = kEps * sqrt((double)n);
  const double floor = 0.01 * kEps * kEps * (double)n * fro2;
  const int sweeps = n > 1 ? cta_jacobi(X, P, n, tol, floor, max_sweeps) : 1;
  if (tid == 0) {
    status[1] = sweeps;
    if (sweeps < 0) atomicOr(status, 2);
  }
  for (int j = warp; j < n; j += (int)(blockDim.x >> 5)) {
    double s2 = 0.0;
    for (int i = lane; i < n; i += 32) s2 += X[i + (size_t)j * n] * X[i + (size_t)j * n];
    s2 = warp_sum(s2);
    if (lane == 0) norms[j] = sqrt(s2);
  }
  for (int e = tid; e < n * n; e += (int)blockDim.x) {
    Yo[e] = X[e];
    Po[e] = P[e];
  }
}

// Out rows of block b ([b L, min(M, (b+1) L))) = Q[rows, :n] * W_b where
// W_b = W[b n : b n + n, :r] (ld ldw).  Grid (nblocks, row chunks).
constexpr int EX_ROWS = 128;
__global__ void __launch_bounds__(256) k_tsqr_expand(int64_t M, int n, int r, int L,
                                                     const double *__restrict__ Q, int64_t ldq,
                                                     const double *__restrict__ W, int64_t ldw,
                                                     double *__restrict__ Out, int64_t ldo) {
  __shared__ double Ws[64][65];
  const int b = blockIdx.x;
  const int64_t r0 = (int64_t)b * L;
  const int mb = (int)min((int64_t)L, M - r0);
  for (int e = threadIdx.x; e < n * r; e += blockDim.x) {
    const int j = e / n, l = e - j * n;
    Ws[l][j] = W[((int64_t)b * n + l) + (int64_t)j * ldw];
  }
  __syncthreads();
  const int c0 = blockIdx.y * EX_ROWS;
  if (c0 >= mb) return;
  const int c1 = min(mb, c0 + EX_ROWS);
  for (int e = threadIdx.x; e < (c1 - c0) * r; e += blockDim.x) {
    const int j = e / (c1 - c0), i = c0 + (e - j * (c1 - c0));
    const double *qi = Q + (r0 + i);
    double acc = 0.0;
    for (int l = 0; l < n; ++l) acc += qi[(int64_t)l * ldq] * Ws[l][j];
    Out[(r0 + i) + (int64_t)j * ldo] = acc;
  }
}

constexpr size_t kSmemCapBytes = 200 * 1024;

int nmax_for(int n) { return n <= 8 ? 8 : n <= 16 ? 16 : n <= 24 ? 24 : n <= 32 ? 32 : n <= 48 ? 48 : 64; }

bool attrs_set = false;
int set_attrs() {
  if (attrs_set) return FTT_OK;
  const int cap = (int)kSmemCapBytes;
  const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
  FTT_CUDA(cudaFuncSetAttribute(k_tsqr_level<8>, a, cap));
  FTT_CUDA(cudaFuncSetAttribute(k_tsqr_level<16>, a, cap));
  FTT_CUDA(cudaFuncSetAttribute(k_tsqr_level<32>, a, cap));
  FTT_CUDA(cudaFuncSetAttribute(k_tsqr_level<24>, a, cap));
  FTT_CUDA(cudaFuncSetAttribute(k_tsqr_level<48>, a, cap));
  FTT_CUDA(cudaFuncSetAttribute(k_tsqr_level<64>, a, cap));
  FTT_CUDA(cudaFuncSetAttribute(k_jacobi_small, a, cap));
  attrs_set = true;
  return FTT_OK;
}

void launch_level(ftt_ctx *ctx, int n, unsigned grid, int64_t M, const double *A, int64_t lda,
                  int trans, double *Rs, int64_t ldr, double *Qo, int64_t ldq, int root,
                  int *status) {
  const int leaf = leaf_rows(n);
  const size_t smem = 8 * (size_t)std::min<int64_t>(M, leaf) * n;
  // a single short block (tree roots, 16..64 rows) runs with just enough
  // warps for its rows and columns: fewer warps per barrier and reduction
  unsigned nt = (unsigned)leaf;
  if (grid == 1) {
    const int64_t need = std::max<int64_t>(std::min<int64_t>(M, leaf), n);
    nt = (unsigned)std::min<int64_t>(leaf, ceil_div(need, 32) * 32);
  }
  switch (nmax_for(n)) {
    case 8:
      k_tsqr_level<8><<<grid, nt, smem, ctx->stream>>>(M, n, A, lda, trans, Rs, ldr, Qo, ldq, root,
                                                         status);
      break;
    case 16:
      k_tsqr_level<16><<<grid, nt, smem, ctx->stream>>>(M, n, A, lda, trans, Rs, ldr, Qo, ldq, root,
                                                          status);
      break;
    case 32:
      k_tsqr_level<32><<<grid, nt, smem, ctx->stream>>>(M, n, A, lda, trans, Rs, ldr, Qo, ldq, root,
                                                          status);
      break;
    case 24:
      k_tsqr_level<24><<<grid, nt, smem, ctx->stream>>>(M, n, A, lda, trans, Rs, ldr, Qo, ldq, root,
                                                          status);
      break;
    case 48:
      k_tsqr_level<48><<<grid, nt, smem, ctx->stream>>>(M, n, A, lda, trans, Rs, ldr, Qo, ldq, root,
                                                          status);
      break;
    default:
      k_tsqr_level<64><<<grid, nt, smem, ctx->stream>>>(M, n, A, lda, trans, Rs, ldr, Qo, ldq, root,
                                                          status);
  }
}

// Levels of the reduction tree for an M x n matrix: rows per level until the
// stack fits the root.
struct Tree {
  std::vector<int64_t> rows;  // rows[0] = M, rows[l+1] = nblocks(l) * n
};

Tree make_tree(int64_t M, int n, int64_t root_rows_max) {
  Tree t;
  t.rows.push_back(M);
  while (t.rows.back() > root_rows_max) t.rows.push_back(ceil_div(t.rows.back(), leaf_rows(n)) * n);
  return t;
}

// Hestenes one-sided Jacobi directly on a short tall block (m x n, n <= 16,
// m * n doubles in shared memory): X P = Y with orthogonal columns; the same
// convergence rule and noise floor as cta_jacobi.  A warp per column pair,
// column length m looped by the lanes.  For the small inner SVDs of the
// low-rank path (B^T, e.g. 512 x 8) this replaces a TSQR tree + Jacobi on R^T
// + Q expansion (5 launches) by one launch.
// wpp warps per column pair: each forms partial dots over its rows, the
// pair's partials are summed in warp order (every warp of the pair gets the
// bitwise same rotation), then each warp rotates its own rows.
__global__ void __launch_bounds__(SVD_NT) k_jacobi_direct(int m, int n, const double *__restrict__ A,
                                                          int64_t lda, int trans, int wpp,
                                                          double *__restrict__ Yo,
                                                          double *__restrict__ Po,
                                                          double *__restrict__ norms,
                                                          int max_sweeps, int *__restrict__ status,
                                                          const double *__restrict__ extra_src,
                                                          double *__restrict__ extra_dst) {
  // status needs no memset: thread 0 writes both words; extra_dst receives
  // *extra_src (a caller's device scalar riding on the same round trip)
  extern __shared__ double S[];  // X m x n (ld m) | P n x n
  __shared__ double red[SVD_NT / 32];
  __shared__ double s_dot[SVD_NT / 32][3];
  __shared__ int s_any;
  double *X = S;
  double *P = S + (size_t)m * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double f = 0.0;
  int bad = 0;
  for (int e = tid; e < m * n; e += (int)blockDim.x) {
    const int j = e / m, i = e - j * m;
    const double v = trans ? A[j + (int64_t)i * lda] : A[i + (int64_t)j * lda];
    bad |= !isfinite(v);
    X[e] = v;
    f += v * v;
  }
  for (int e = tid; e < n * n; e += (int)blockDim.x) P[e] = (e / n == e % n) ? 1.0 : 0.0;
  if (tid == 0 && extra_src) *extra_dst = *extra_src;
  if (__syncthreads_or(bad)) {
    if (tid == 0) {
      status[0] = 1;
      status[1] = 0;
    }
    return;
  }
  const double fro2 = cta_sum(f, red);
  const double tol = kEps * sqrt((double)n);
  const double floor = 0.01 * kEps * kEps * (double)m * fro2;
  const int ne = n + (n & 1), npairs = ne / 2;
  const int pi = warp / wpp, sub = warp - pi * wpp;  // nw == npairs * wpp
  int sweeps = -1;
  for (int sw = 0; sw < max_sweeps && n > 1; ++sw) {
    if (tid == 0) s_any = 0;
    __syncthreads();
    for (int round = 0; round < ne - 1; ++round) {
      int p, q;
      rr_pair(ne, round, pi, &p, &q);
      const bool live = pi < npairs && p < n && q < n;
      double *xp = X + (size_t)(live ? p : 0) * m, *xq = X + (size_t)(live ? q : 0) * m;
      if (live) {
        double a = 0.0, b = 0.0, g = 0.0;
        for (int i = sub * 32 + lane; i < m; i += 32 * wpp) {
          const double u = xp[i], v = xq[i];
          a += u * u;
          b += v * v;
          g += u * v;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        if (lane == 0) {
          s_dot[warp][0] = a;
          s_dot[warp][1] = b;
          s_dot[warp][2] = g;
        }
      }
      __syncthreads();
      if (live) {
        double a = 0.0, b = 0.0, g = 0.0;
        for (int w = pi * wpp; w < pi * wpp + wpp; ++w) {
          a += s_dot[w][0];
          b += s_dot[w][1];
          g += s_dot[w][2];
        }
        if (a > floor && b > floor && fabs(g) > tol * sqrt(a * b)) {
          const double zeta = (b - a) / (2.0 * g);
          const double t = copysign(1.0 / (fabs(zeta) + sqrt(1.0 + zeta * zeta)), zeta);
          const double c = rsqrt(1.0 + t * t);
          const double sn = c * t;
          for (int i = sub * 32 + lane; i < m; i += 32 * wpp) {
            const double u = xp[i], v = xq[i];
            xp[i] = c * u - sn * v;
            xq[i] = sn * u + c * v;
          }
          if (sub == 0) {
            double *pp = P + (size_t)p * n, *pq = P + (size_t)q * n;
            if (lane < n) {
              const double pu = pp[lane], pv = pq[lane];
              pp[lane] = c * pu - sn * pv;
              pq[lane] = sn * pu + c * pv;
            }
            if (lane == 0) s_any = 1;
          }
        }
      }
      __syncthreads();
    }
    if (!s_any) {
      sweeps = sw + 1;
      break;
    }
    __syncthreads();
  }
  if (n <= 1) sweeps = 1;
  if (tid == 0) {
    status[0] = sweeps < 0 ? 2 : 0;
    status[1] = sweeps;
  }
  for (int j = warp; j < n; j += nw) {
    double s2 = 0.0;
    for (int i = lane; i < m; i += 32) s2 += X[i + (size_t)j * m] * X[i + (size_t)j * m];
    s2 = warp_sum(s2);
    if (lane == 0) norms[j] = sqrt(s2);
  }
  for (int e = tid; e < m * n; e += (int)blockDim.x) Yo[e] = X[e];
  for (int e = tid; e < n * n; e += (int)blockDim.x) Po[e] = P[e];
}

// The same factorisation for a short tall block (m x n, n <= 16) with the
// rotations chosen on R instead of on X: X = Q R (Householder in shared
// memory, a warp per column for the dots, 2 barriers per column), one-sided
// Jacobi R P = Y_R by ONE warp without CTA barriers (4 lanes per column
// pair, 8 pairs per round; the dots are over n rows instead of m), then
// Y = Q [Y_R; 0] (the reflectors in reverse).  Same outputs, convergence rule
// and noise floor (m of X) as k_jacobi_direct; X P = Q R P = Y.
constexpr int QJ_NT = 512;
__global__ void __launch_bounds__(QJ_NT) k_jacobi_qr(int m, int n, const double *__restrict__ A,
                                                     int64_t lda, int trans,
                                                     double *__restrict__ Yo,
                                                     double *__restrict__ Po,
                                                     double *__restrict__ norms, int max_sweeps,
                                                     int *__restrict__ status,
                                                     const double *__restrict__ extra_src,
                                                     double *__restrict__ extra_dst) {
  extern __shared__ double S[];  // X m x n | Y m x n | R n x n | P n x n (all col-major)
  __shared__ double red[QJ_NT / 32];
  __shared__ double s_dot[16];
  __shared__ double s_tau[16];
  __shared__ int s_sweeps;
  double *X = S, *Y = S + (size_t)m * n, *R = Y + (size_t)m * n, *P = R + n * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double f = 0.0;
  int bad = 0;
  for (int e = tid; e < m * n; e += QJ_NT) {
    const int j = e / m, i = e - j * m;
    const double v = trans ? A[j + (int64_t)i * lda] : A[i + (int64_t)j * lda];
    bad |= !isfinite(v);
    X[e] = v;
    f += v * v;
  }
  if (tid == 0 && extra_src) *extra_dst = *extra_src;
  if (__syncthreads_or(bad)) {
    if (tid == 0) {
      status[0] = 1;
      status[1] = 0;
    }
    return;
  }
  const double fro2 = cta_sum(f, red);
  // ---- Householder QR: column j's reflector v = [1; x_j(j+1:) / v0]
  __shared__ double s_w[16];
  for (int j = 0; j < n; ++j) {
    // warp w: column c = j + w; every warp also forms |x_j(j+1:)|^2 itself
    // (same order in every warp: bitwise the same tau), then w_c =
    // tau (x_jc + (x_j . x_c) / v0) before anything is updated
    const int c = j + warp;
    double tau = 0.0, beta = 0.0, v0 = 1.0;
    if (c < n) {
      const double *xj = X + (size_t)j * m, *xc = X + (size_t)c * m;
      double d = 0.0, sub = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) {
        const double u = xj[i];
        d += u * xc[i];
        sub += u * u;
      }
      d = warp_sum(d);
      sub = warp_sum(sub);
      const double alpha = xj[j];
      beta = alpha;
      if (sub > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + sub), alpha);
        v0 = alpha - beta;
        tau = (beta - alpha) / beta;
      }
      if (lane == 0) {
        s_w[warp] = tau * (xc[j] + d / v0);
        if (warp == 0) {
          s_tau[j] = tau;
          s_dot[0] = beta;
          s_dot[1] = v0;
        }
      }
    }
    __syncthreads();
    tau = s_tau[j];
    v0 = s_dot[1];
    if (tau != 0.0) {
      const double inv = 1.0 / v0;
      const int nc = n - j - 1, mr = m - j;
      for (int e = tid; e < nc * mr; e += QJ_NT) {
        const int k = e / mr, i = j + (e - k * mr), cc = j + 1 + k;
        X[i + (size_t)cc * m] -= s_w[k + 1] * (i == j ? 1.0 : X[i + (size_t)j * m] * inv);
      }
    }
    __syncthreads();
    if (tau != 0.0) {
      const double inv = 1.0 / v0;
      for (int i = j + 1 + tid; i < m; i += QJ_NT) X[i + (size_t)j * m] *= inv;
    }
    if (tid == 0) X[j + (size_t)j * m] = s_dot[0];
    // the next step's dots read columns > j only, and its barrier orders
    // these writes before column j is read again
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += QJ_NT) {
    const int b = e / n, a = e - b * n;
    R[e] = a <= b ? X[a + (size_t)b * m] : 0.0;
    P[e] = a == b ? 1.0 : 0.0;
  }
  __syncthreads();
  // ---- one-sided Jacobi on R by warp 0: pair g = lane / 4, rows lane % 4 + 4 k
  if (warp == 0) {
    const double tol = kEps * sqrt((double)n);
    const double floor = 0.01 * kEps * kEps * (double)m * fro2;
    const int ne = n + (n & 1), g = lane >> 2, sl = lane & 3;
    int sweeps = -1;
    for (int sw = 0; sw < max_sweeps && n > 1; ++sw) {
      int any = 0;
      for (int round = 0; round < ne - 1; ++round) {
        int p = 0, q = 0;
        const bool live = g < ne / 2;
        if (live) rr_pair(ne, round, g, &p, &q);
        const bool ok = live && p < n && q < n;
        double *rp = R + (size_t)(ok ? p : 0) * n, *rq = R + (size_t)(ok ? q : 0) * n;
        double a = 0.0, b = 0.0, gg = 0.0;
        if (ok)
          for (int i = sl; i < n; i += 4) {
            const double u = rp[i], v = rq[i];
            a += u * u;
            b += v * v;
            gg += u * v;
          }
        // sum over the pair's 4 lanes (xor 1, 2: bitwise the same in all 4)
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          gg += __shfl_xor_sync(0xffffffffu, gg, o);
        }
        // the same test and angle as the other Jacobi kernels with two fewer
        // fp64 sqrt/div on the warp's serial chain: |g| > tol sqrt(ab) as
        // g^2 > tol^2 ab, and t = sgn(d) 2g / (|d| + sqrt(d^2 + 4 g^2)),
        // d = b - a (= sgn(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = d / 2g)
        if (ok && a > floor && b > floor && gg * gg > tol * tol * (a * b)) {
          const double dd = b - a;
          const double t = copysign(1.0, dd) * (2.0 * gg) / (fabs(dd) + sqrt(dd * dd + 4.0 * gg * gg));
          const double cs = rsqrt(1.0 + t * t);
          const double sn = cs * t;
          double *pp = P + (size_t)p * n, *pq = P + (size_t)q * n;
          for (int i = sl; i < n; i += 4) {
            const double u = rp[i], v = rq[i];
            rp[i] = cs * u - sn * v;
            rq[i] = sn * u + cs * v;
            const double pu = pp[i], pv = pq[i];
            pp[i] = cs * pu - sn * pv;
            pq[i] = sn * pu + cs * pv;
          }
          any = 1;
        }
        __syncwarp();
      }
      if (!__any_sync(0xffffffffu, any)) {
        sweeps = sw + 1;
        break;
      }
    }
    if (n <= 1) sweeps = 1;
    if (lane == 0) s_sweeps = sweeps;
  }
  __syncthreads();
  // ---- Y = Q [Y_R; 0]: H_{n-1} first, H_0 last
  for (int e = tid; e < m * n; e += QJ_NT) {
    const int c = e / m, i = e - c * m;
    Y[e] = i < n ? R[i + c * n] : 0.0;
  }
  __syncthreads();
  for (int j = n - 1; j >= 0; --j) {
    const double tau = s_tau[j];
    if (tau == 0.0) continue;  // uniform: s_tau is shared
    const int c = warp;
    if (c < n) {
      const double *v = X + (size_t)j * m, *yc = Y + (size_t)c * m;
      double d = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) d += v[i] * yc[i];
      d = warp_sum(d);
      if (lane == 0) s_dot[c] = tau * (yc[j] + d);
    }
    __syncthreads();
    for (int e = tid; e < n * (m - j); e += QJ_NT) {
      const int cc = e / (m - j), i = j + e % (m - j);
      Y[i + (size_t)cc * m] -= s_dot[cc] * (i == j ? 1.0 : X[i + (size_t)j * m]);
    }
    __syncthreads();
  }
  if (tid == 0) {
    status[0] = s_sweeps < 0 ? 2 : 0;
    status[1] = s_sweeps;
  }
  for (int j = warp; j < n; j += QJ_NT / 32) {
    double s2 = 0.0;
    for (int i = lane; i < n; i += 32) s2 += R[i + (size_t)j * n] * R[i + (size_t)j * n];
    s2 = warp_sum(s2);
    if (lane == 0) norms[j] = sqrt(s2);
  }
  for (int e = tid; e < m * n; e += QJ_NT) Yo[e] = Y[e];
  for (int e = tid; e < n * n; e += QJ_NT) Po[e] = P[e];
}

}  // namespace

bool tsqr_ok(int64_t m, int64_t n) { return n >= 1 && n <= 64 && m >= n; }

// Reduce A_tall (M x n) level by level (Q factors kept in qs[2 l], stacked R
// in qs[2 l + 1]) until the root fits.
static int tsqr_reduce(ftt_ctx *ctx, int64_t M, int n, const double *A, int64_t lda, int trans,
                       int64_t root_rows_max, Tree *tree, std::vector<double *> *qs,
                       const double **root, int64_t *root_ld, int *status) {
  *tree = make_tree(M, n, root_rows_max);
  const Tree &t = *tree;
  const double *cur = A;
  int64_t cur_ld = lda;
  int cur_trans = trans;
  for (size_t l = 0; l + 1 < t.rows.size(); ++l) {
    const int64_t Ml = t.rows[l];
    const int64_t nb = ceil_div(Ml, leaf_rows(n));
    double *Qo = nullptr, *Rs = nullptr;
    FTT_CHECK(owned_alloc(ctx, (void **)&Qo, 8 * (size_t)Ml * n));
    FTT_CHECK(owned_alloc(ctx, (void **)&Rs, 8 * (size_t)t.rows[l + 1] * n));
    launch_level(ctx, n, (unsigned)nb, Ml, cur, cur_ld, cur_trans, Rs, t.rows[l + 1], Qo, Ml, 0,
                 status);
    FTT_LAUNCHED(ctx);
    qs->push_back(Qo);
    qs->push_back(Rs);
    cur = Rs;
    cur_ld = t.rows[l + 1];
    cur_trans = 0;
  }
  *root = cur;
  *root_ld = cur_ld;
  return FTT_OK;
}

// Expand W (root rows x r) back down the tree into Out (M x r).
static int tsqr_expand(ftt_ctx *ctx, const Tree &t, int n, int r, const std::vector<double *> &qs,
                       const double *W, int64_t ldw, double *Out, int64_t ldo) {
  const int nl = (int)t.rows.size() - 1;
  const double *cur = W;
  int64_t cur_ld = ldw;
  std::vector<double *> tmp;
  for (int l = nl - 1; l >= 0; --l) {
    const int64_t Ml = t.rows[l];
    const int leaf = leaf_rows(n);
    const int64_t nb = ceil_div(Ml, leaf);
    double *dst = Out;
    int64_t dld = ldo;
    if (l > 0) {
      FTT_CHECK(owned_alloc(ctx, (void **)&dst, 8 * (size_t)Ml * r));
      dld = Ml;
      tmp.push_back(dst);
    }
    dim3 grid((unsigned)nb, (unsigned)ceil_div(leaf, EX_ROWS));
    k_tsqr_expand<<<grid, 256, 0, ctx->stream>>>(Ml, n, r, leaf, qs[2 * l], Ml, cur, cur_ld, dst,
                                                 dld);
    FTT_LAUNCHED(ctx);
    cur = dst;
    cur_ld = dld;
  }
  for (double *p : tmp) owned_free(ctx, p);
  return FTT_OK;
}

int tsqr_q(ftt_ctx *ctx, int64_t M, int64_t n64, const double *A, int64_t lda, int trans,
           double *Q, int64_t ldq, double *R, int64_t ldr, bool check) {
  const int n = (int)n64;
  FTT_CHECK(set_attrs());
  // deferred mode: flags go to the context's sticky word (no round trip)
  const bool deferred = check && ctx->defer_checks;
  int *status = nullptr;
  if (deferred) {
    status = ctx->sticky;
  } else {
    FTT_CHECK(owned_alloc(ctx, (void **)&status, 64));
    FTT_CUDA(cudaMemsetAsync(status, 0, 64, ctx->stream));
  }
  Tree t;
  std::vector<double *> qs;
  const double *root;
  int64_t root_ld;
  FTT_CHECK(tsqr_reduce(ctx, M, n, A, lda, trans, leaf_rows(n), &t, &qs, &root, &root_ld, status));
  const int64_t Mr = t.rows.back();
  if (t.rows.size() == 1) {
    launch_level(ctx, n, 1, Mr, root, root_ld, trans, R, ldr, Q, ldq, 1, status);
    FTT_LAUNCHED(ctx);
  } else {
    double *Qr = nullptr;
    FTT_CHECK(owned_alloc(ctx, (void **)&Qr, 8 * (size_t)Mr * n));
    launch_level(ctx, n, 1, Mr, root, root_ld, 0, R, ldr, Qr, Mr, 1, status);
    FTT_LAUNCHED(ctx);
    FTT_CHECK(tsqr_expand(ctx, t, n, n, qs, Qr, Mr, Q, ldq));
    owned_free(ctx, Qr);
  }
  for (double *p : qs) owned_free(ctx, p);
  int h = 0;
  if (deferred) return FTT_OK;
  if (check) FTT_CHECK(copy_to_host(ctx, &h, status, sizeof(int)));
  owned_free(ctx, status);
  if (h & 1) {
    set_error("matrix entries must be finite");
    return FTT_ERR_NONFINITE;
  }
  return FTT_OK;
}

int tsqr_svd(ftt_ctx *ctx, int64_t M, int64_t n64, const double *A, int64_t lda, int trans,
             double *U, int64_t ldu, double *Y, double *norms_host, int *sweeps,
             const double *extra_dev, double *extra_host) {
  const int n = (int)n64;
  FTT_CHECK(set_attrs());
  // status (2 ints) | norms n | R n x n | P n x n
  double *dev = nullptr;
  // status (2 ints) | extra | norms n | R n x n | P n x n
  FTT_CHECK(owned_alloc(ctx, (void **)&dev, 8 * (size_t)(2 + n + 2 * (size_t)n * n)));
  int *status = reinterpret_cast<int *>(dev);
  double *norms = dev + 2;
  double *R = norms + n;
  double *P = R + (size_t)n * n;
  FTT_CUDA(cudaMemsetAsync(status, 0, 16, ctx->stream));
  Tree t;
  std::vector<double *> qs;
  const double *root;
  int64_t root_ld;
  FTT_CHECK(tsqr_reduce(ctx, M, n, A, lda, trans, leaf_rows(n), &t, &qs, &root, &root_ld, status));
  const int64_t Mr = t.rows.back();
  const bool single = t.rows.size() == 1;
  double *Qr = nullptr, *W = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&Qr, 8 * (size_t)Mr * n));
  launch_level(ctx, n, 1, Mr, root, root_ld, single ? trans : 0, R, n, Qr, Mr, 1, status);
  FTT_LAUNCHED(ctx);
  const int max_sweeps = 60;
  // one warp per column pair of a round: small n needs few warps (and gets
  // cheaper barriers)
  const int jt = 32 * std::max(1, std::min(SVD_NT / 32, (n + 1) / 2));
  k_jacobi_small<<<1, jt, 16 * (size_t)n * n, ctx->stream>>>(n, R, n, Y, P, norms, max_sweeps,
                                                              status);
  FTT_LAUNCHED(ctx);
  // W = Q_root P, then down the tree
  if (!single) FTT_CHECK(owned_alloc(ctx, (void **)&W, 8 * (size_t)Mr * n));
  {
    dim3 grid(1, (unsigned)ceil_div(Mr, EX_ROWS));
    k_tsqr_expand<<<grid, 256, 0, ctx->stream>>>(Mr, n, n, (int)Mr, Qr, Mr, P, n, single ? U : W,
                                                 single ? ldu : Mr);
    FTT_LAUNCHED(ctx);
  }
  if (!single) FTT_CHECK(tsqr_expand(ctx, t, n, n, qs, W, Mr, U, ldu));
  owned_free(ctx, Qr);
  if (W) owned_free(ctx, W);
  for (double *p : qs) owned_free(ctx, p);
  // one round trip: status, the caller's device scalar and the norms
  if (extra_dev)
    FTT_CUDA(cudaMemcpyAsync(dev + 1, extra_dev, sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
  std::vector<double> h(n + 2);
  FTT_CHECK(copy_to_host(ctx, h.data(), dev, 8 * (size_t)(n + 2)));
  if (extra_dev && extra_host) *extra_host = h[1];
  owned_free(ctx, dev);
  int st[2];
  memcpy(st, h.data(), 8);
  if (st[0] & 1) {
    set_error("matrix entries must be finite");
    return FTT_ERR_NONFINITE;
  }
  if (st[0] & 2) {
    set_error("Jacobi SVD did not converge in %d sweeps", max_sweeps);
    return FTT_ERR_NOCONV;
  }
  if (sweeps) *sweeps = st[1];
  memcpy(norms_host, h.data() + 2, 8 * (size_t)n);
  return FTT_OK;
}

bool direct_small_ok(int64_t m, int64_t n) {
  static const bool off = getenv("FTT_NO_DIRECT_SMALL") != nullptr;
  return !off && n >= 1 && n <= 16 && m >= n && m * n * 8 <= 160 * 1024;
}

// One-sided Jacobi directly on the short tall A_tall (m x n): Y = A_tall P
// (m x n, ld m), P (n x n), norms_host[j] = ||Y_j|| (unsorted).
int direct_small_svd(ftt_ctx *ctx, int64_t m, int64_t n, const double *A, int64_t lda, int trans,
                     double *Y, double *P, double *norms_host, int *sweeps,
                     const double *extra_dev, double *extra_host) {
  static bool attr = false;
  if (!attr) {
    FTT_CUDA(cudaFuncSetAttribute(k_jacobi_direct, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024));
    attr = true;
  }
  double *dev = nullptr;  // status (2 ints) | pad | norms n
  FTT_CHECK(owned_alloc(ctx, (void **)&dev, 8 * (size_t)(2 + n)));
  int *status = reinterpret_cast<int *>(dev);
  // warps per pair: enough that each lane holds <= ~8 rows, <= SVD_NT total
  static const int wpp_env = getenv("FTT_DIRECT_WPP") ? atoi(getenv("FTT_DIRECT_WPP")) : 0;
  const int npairs = (int)((n + 1) / 2);
  int wpp = wpp_env > 0 ? wpp_env : (int)std::min<int64_t>(8, std::max<int64_t>(1, ceil_div(m, 256)));
  wpp = std::max(1, std::min(wpp, SVD_NT / 32 / std::max(1, npairs)));
  const int jt = 32 * std::max(1, npairs) * wpp;
  const int max_sweeps = 60;
  static const bool qr_off = getenv("FTT_NO_QR_JACOBI") != nullptr;
  const size_t qj_smem = 8 * (size_t)(2 * m * n + 2 * n * n);
  if (!qr_off && n <= 16 && qj_smem <= 200 * 1024) {
    static bool qattr = false;
    if (!qattr) {
      FTT_CUDA(cudaFuncSetAttribute(k_jacobi_qr, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    200 * 1024));
      qattr = true;
    }
    k_jacobi_qr<<<1, QJ_NT, qj_smem, ctx->stream>>>((int)m, (int)n, A, lda, trans, Y, P, dev + 2,
                                                    max_sweeps, status, extra_dev, dev + 1);
  } else {
    k_jacobi_direct<<<1, jt, 8 * (size_t)(m * n + n * n), ctx->stream>>>(
        (int)m, (int)n, A, lda, trans, wpp, Y, P, dev + 2, max_sweeps, status, extra_dev, dev + 1);
  }
  FTT_LAUNCHED(ctx);
  std::vector<double> h(n + 2);
  FTT_CHECK(copy_to_host(ctx, h.data(), dev, 8 * (size_t)(n + 2)));
  if (extra_dev && extra_host) *extra_host = h[1];
  owned_free(ctx, dev);
  int st[2];
  memcpy(st, h.data(), 8);
  if (st[0] & 1) {
    set_error("matrix entries must be finite");
    return FTT_ERR_NONFINITE;
  }
  if (st[0] & 2) {
    set_error("Jacobi SVD did not converge in %d sweeps", max_sweeps);
    return FTT_ERR_NOCONV;
  }
  if (sweeps) *sweeps = st[1];
  static const bool debug = getenv("FTT_DEBUG") != nullptr;
  if (debug) fprintf(stderr, "[ftt] direct small svd m=%lld n=%lld sweeps %d\n", (long long)m,
                     (long long)n, st[1]);
  memcpy(norms_host, h.data() + 2, 8 * (size_t)n);
  return FTT_OK;
}

}  // namespace ftt
