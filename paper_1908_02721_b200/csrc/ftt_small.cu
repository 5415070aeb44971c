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

// ---- several rows per thread (n <= 16) --------------------------------
// The one-row-per-thread kernels above spend each column step on a CTA-wide
// reduce-scatter of n partial dots: with 512 threads that is 16 warps x 31
// fp64 shuffles per step (the shuffle unit serialises ~1 warp-shuffle per
// clock), so a 512 x 16 leaf took ~53 us and a leaf level ran one CTA per SM.
// Here a thread owns RPT rows (i = threadIdx.x + r * blockDim.x, coalesced),
// sums its rows' products locally first, and the warp reduce-scatter halves
// from the first stage (16 shuffles for 16 slots): 4x fewer warps per step,
// ~2x fewer shuffles per warp, and a 512-row leaf is a 128-thread CTA that
// shares its SM with others.

// W slots over 32 lanes by recursive halving: at offset s = 16, 8, ...
// each lane keeps the half of its live slots selected by its lane bit and
// adds the partner's copy; once one slot is left the remaining offsets add
// whole values.  Lane l ends with the warp total of slot (l >> (5 - log2 W))
// (all lanes of a slot hold the same bits: fp add commutes).
template <int W>
__device__ __forceinline__ double rs_halving(double (&v)[32], int lane) {
  int live = W;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    if (live > 1) {
      const int h = live / 2;
      const bool upper = (lane & s) != 0;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < h) {
          const double send = upper ? v[j] : v[j + h];
          const double keep = upper ? v[j + h] : v[j];
          v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
      live = h;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], s);
    }
  }
  return v[0];
}
template <int W>
__device__ __forceinline__ int rs_slot(int lane) {
  constexpr int sh = W >= 32 ? 0 : (W >= 16 ? 1 : (W >= 8 ? 2 : (W >= 4 ? 3 : (W >= 2 ? 4 : 5))));
  return (lane >> sh) & (W - 1);
}
template <int W>
__device__ __forceinline__ bool rs_writer(int lane) {
  constexpr int sh = W >= 32 ? 0 : (W >= 16 ? 1 : (W >= 8 ? 2 : (W >= 4 ? 3 : (W >= 2 ? 4 : 5))));
  return (lane & ((1 << sh) - 1)) == 0;
}

// red[warp][u] = sum over the warp's rows of x_r * b[r][u] (u < NMAX <= 16)
template <int NMAX, int RPT>
__device__ __forceinline__ void rows_partials(double (*red)[NMAX], const double (&x)[RPT],
                                              const double (&b)[RPT][NMAX]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double p[32];
#pragma unroll
  for (int u = 0; u < 32; ++u) p[u] = 0.0;
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int u = 0; u < NMAX; ++u) p[u] = fma(x[r], b[r][u], p[u]);
  const double tot = rs_halving<NMAX>(p, lane);
  if (rs_writer<NMAX>(lane)) red[warp][rs_slot<NMAX>(lane)] = tot;
}

// reg_qr for RPT rows per thread (row i = threadIdx.x + r blockDim.x; the
// pivot rows c < n <= 16 are slot 0 of threads c).  Same outputs as reg_qr.
template <int NMAX, int RPT>
__device__ void reg_qr_m(double (&a)[RPT][NMAX], int m, int n, double *Sref, Scratch<NMAX> &sc) {
  const int t = threadIdx.x, T = blockDim.x;
  const int k = min(m, n);
  for (int c = 0; c < k; ++c) {
    const int nc = n - c;
    if (t == c) {
#pragma unroll
      for (int u = 0; u < NMAX; ++u) sc.rowc[u] = a[0][u];
    }
    double x[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = t + r * T;
      x[r] = (i > c && i < m) ? a[r][0] : 0.0;
    }
    rows_partials<NMAX, RPT>(sc.red, x, a);
    __syncthreads();
    if (t < nc) {  // thread u: column c + u (u = 0: the pivot's scalars)
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
      if (t == 0) {
        sc.tau[c] = tau;
        sc.beta[c] = beta;
        sc.sc[0] = tau;
        sc.sc[1] = beta;
        sc.sc[2] = scal;
      } else {
        sc.wv[t] = tau * (sc.rowc[t] + scal * sum_warps<NMAX>(sc.red, t));
      }
    } else if (t < NMAX) {
      sc.wv[t] = 0.0;  // columns past n - c do not move
    }
    __syncthreads();
    const double tau = sc.sc[0], beta = sc.sc[1], scal = sc.sc[2];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = t + r * T;
      if (i > c && i < m) {
        const double v = scal * a[r][0];
        if (tau != 0.0) {
#pragma unroll
          for (int u = 1; u < NMAX; ++u) a[r][u] = fma(-sc.wv[u], v, a[r][u]);
        }
        a[r][0] = v;
      } else if (i == c) {
        if (tau != 0.0) {
#pragma unroll
          for (int u = 1; u < NMAX; ++u) a[r][u] -= sc.wv[u];
        }
        a[r][0] = beta;
      }
      if (i < m) Sref[i + (size_t)c * m] = a[r][0];
#pragma unroll
      for (int u = 0; u + 1 < NMAX; ++u) a[r][u] = a[r][u + 1];
      a[r][NMAX - 1] = 0.0;
    }
  }
  __syncthreads();
}

// z <- Q z (apply_q) for RPT rows per thread.
template <int NMAX, int RPT>
__device__ void apply_q_m(const double *Sref, const double *tau_s, double (&z)[RPT][NMAX], int m,
                          int k, int ncol, Scratch<NMAX> &sc) {
  const int t = threadIdx.x, T = blockDim.x;
  for (int c = k - 1; c >= 0; --c) {
    const double tau = tau_s[c];
    if (tau == 0.0) continue;
    double v[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = t + r * T;
      v[r] = i == c ? 1.0 : ((i > c && i < m) ? Sref[i + (size_t)c * m] : 0.0);
    }
    rows_partials<NMAX, RPT>(sc.red, v, z);
    __syncthreads();
    if (t < ncol) sc.wv[t] = tau * sum_warps<NMAX>(sc.red, t);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int u = 0; u < NMAX; ++u)
        if (u < ncol) z[r][u] = fma(-sc.wv[u], v[r], z[r][u]);
  }
  __syncthreads();
}

template <int NMAX, int RPT>
__device__ bool load_rows(double (&a)[RPT][NMAX], int mb, int n, const double *__restrict__ buf,
                          int64_t ld, int trans, int64_t r0) {
  int bad = 0;
  const int t = threadIdx.x, T = blockDim.x;
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = t + r * T;
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
      double v = 0.0;
      if (i < mb && j < n) v = trans ? buf[j + (r0 + i) * ld] : buf[(r0 + i) + (int64_t)j * ld];
      bad |= !isfinite(v);
      a[r][j] = v;
    }
  }
  return !__syncthreads_or(bad);
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

// One-sided Jacobi on X (n x n, n <= NM <= 16, ld ldx) accumulating P (ld
// ldp), both in shared memory, run by ONE warp out of registers: lane c < 16
// holds column c of X, lane 16 + c column c of P.  Round r of the circle
// method pairs column c with (2 r - c) mod (ne - 1) (column ne - 1 with r),
// so each lane finds its partner arithmetically and one shuffle per element
// brings the partner's column (X and P lanes in the same instruction).  Both
// lanes of a pair form the same dots in the same order (bit-identical
// decision and angle); the P lanes then fetch their column's rotation.  No
// shared memory or barriers inside the sweep: the smem variants spent most
// of their time on bank conflicts (all columns of an n = 16 block start in
// the same bank) and on the serial fp64 div/sqrt chain, here one sqrt and one
// rsqrt per round:
//   r = sqrt(d^2 + 4 g^2), w = |d| + r, rho = rsqrt(w^2 + 4 g^2),
//   c = w rho, s = sgn(d) 2 g rho      (d = |x_q|^2 - |x_p|^2, g = x_p . x_q)
// which is the same rotation as t = sgn(d) 2g / (|d| + r), c = 1/sqrt(1+t^2).
// Convergence rule as cta_jacobi.  Writes X and P back; returns the sweeps
// used (-1 if max_sweeps was exhausted).  Call from one full warp.
template <int NM>
__device__ int warp_jacobi_cols(double *X, int ldx, double *P, int ldp, int n, double tol,
                                double floor, int max_sweeps) {
  static_assert(NM <= 16, "one lane per column, P in the upper half-warp");
  const int lane = threadIdx.x & 31, c = lane & 15;
  const bool isP = lane >= 16;
  double x[NM];
#pragma unroll
  for (int i = 0; i < NM; ++i)
    x[i] = (c < n && i < n) ? (isP ? P[i + c * ldp] : X[i + c * ldx]) : 0.0;
  const int ne = n + (n & 1), L = ne - 1;
  const double tol2 = tol * tol;
  int sweeps = n > 1 ? -1 : 1;
  for (int sw = 0; sw < max_sweeps && n > 1; ++sw) {
    int any = 0;
    for (int round = 0; round < L; ++round) {
      int pa;
      if (c == L) pa = round;
      else if (c == round) pa = L;
      else {
        pa = 2 * round - c;
        pa = pa < 0 ? pa + L : (pa >= L ? pa - L : pa);
      }
      const bool live = c < n && pa < n;
      const bool first = c < pa;
      const int src = (lane & 16) | (pa & 15);
      // |own column|^2 (4 chains), then the partner's column and its norm:
      // both lanes of a pair hold the same a = |x_p|^2, b = |x_q|^2 bits
      double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;
#pragma unroll
      for (int i = 0; i < NM; i += 4) {
        q0 = fma(x[i], x[i], q0);
        if (i + 1 < NM) q1 = fma(x[i + 1], x[i + 1], q1);
        if (i + 2 < NM) q2 = fma(x[i + 2], x[i + 2], q2);
        if (i + 3 < NM) q3 = fma(x[i + 3], x[i + 3], q3);
      }
      const double sx = (q0 + q1) + (q2 + q3);
      double y[NM];
#pragma unroll
      for (int i = 0; i < NM; ++i) y[i] = __shfl_sync(0xffffffffu, x[i], src);
      const double sy = __shfl_sync(0xffffffffu, sx, src);
      double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
#pragma unroll
      for (int i = 0; i < NM; i += 4) {
        g0 = fma(x[i], y[i], g0);
        if (i + 1 < NM) g1 = fma(x[i + 1], y[i + 1], g1);
        if (i + 2 < NM) g2 = fma(x[i + 2], y[i + 2], g2);
        if (i + 3 < NM) g3 = fma(x[i + 3], y[i + 3], g3);
      }
      const double g = (g0 + g1) + (g2 + g3);
      const double a = first ? sx : sy, b = first ? sy : sx;
      int rot = (!isP && live && a > floor && b > floor && g * g > tol2 * (a * b)) ? 1 : 0;
      double cs = 1.0, sn = 0.0;
      if (rot) {
        const double dd = b - a, gd = 2.0 * g;
        const double r = sqrt(fma(dd, dd, gd * gd));
        const double w = fabs(dd) + r;
        const double rho = rsqrt(fma(w, w, gd * gd));
        cs = w * rho;
        sn = copysign(1.0, dd) * gd * rho;
      }
      const double pcs = __shfl_sync(0xffffffffu, cs, c), psn = __shfl_sync(0xffffffffu, sn, c);
      const int prot = __shfl_sync(0xffffffffu, rot, c);
      if (isP) {
        cs = pcs;
        sn = psn;
        rot = prot;
      }
      if (rot) {
        // x_p <- c x_p - s x_q ,  x_q <- c x_q + s x_p
        const double s2 = first ? -sn : sn;
#pragma unroll
        for (int i = 0; i < NM; ++i) x[i] = fma(cs, x[i], s2 * y[i]);
      }
      any |= rot;
    }
    if (!__any_sync(0xffffffffu, any)) {
      sweeps = sw + 1;
      break;
    }
  }
  if (c < n) {
#pragma unroll
    for (int i = 0; i < NM; ++i)
      if (i < n) {
        if (isP) P[i + c * ldp] = x[i];
        else X[i + c * ldx] = x[i];
      }
  }
  __syncwarp();
  return sweeps;
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

// k_tsqr_level for n <= 16 with RPT rows per thread (leaf = blockDim * RPT
// rows; same outputs).
constexpr int LEAF_RPT = 2;
template <int NMAX, int RPT>
__global__ void __launch_bounds__(LEAF_MAX / RPT) k_tsqr_level_m(
    int64_t M, int n, const double *__restrict__ A, int64_t lda, int trans, double *__restrict__ Rs,
    int64_t ldr, double *__restrict__ Qo, int64_t ldq, int root, int *__restrict__ status) {
  extern __shared__ double Sref[];
  __shared__ Scratch<NMAX> sc;
  const int T = blockDim.x, t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * T * RPT;
  const int mb = (int)min((int64_t)T * RPT, M - r0);
  const int k = min(mb, n);
  double a[RPT][NMAX];
  if (!load_rows<NMAX, RPT>(a, mb, n, A, lda, trans, r0)) {
    if (t == 0) atomicOr(status, 1);
    return;
  }
  reg_qr_m<NMAX, RPT>(a, mb, n, Sref, sc);
#pragma unroll
  for (int r = 0; r < RPT; ++r) {  // columns k.. (only when the block is wider than tall)
    const int i = t + r * T;
    if (i < mb) {
#pragma unroll
      for (int u = 0; u < NMAX; ++u)
        if (k + u < n) Sref[i + (size_t)(k + u) * mb] = a[r][u];
    }
  }
  __syncthreads();
  if (Rs && t < n) {  // row t of R_b (sign-fixed at the root)
    const double sg = (root && t < k && sc.beta[t] < 0.0) ? -1.0 : 1.0;
    const int64_t rb = (int64_t)blockIdx.x * n + t;
    for (int j = 0; j < n; ++j)
      Rs[rb + (int64_t)j * ldr] = (t <= j && t < mb) ? sg * Sref[t + (size_t)j * mb] : 0.0;
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = t + r * T;
#pragma unroll
    for (int j = 0; j < NMAX; ++j) a[r][j] = (i == j && j < k) ? 1.0 : 0.0;
  }
  apply_q_m<NMAX, RPT>(Sref, sc.tau, a, mb, k, k, sc);
  double sg[NMAX];
#pragma unroll
  for (int j = 0; j < NMAX; ++j) sg[j] = j < k ? ((root && sc.beta[j] < 0.0) ? -1.0 : 1.0) : 0.0;
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = t + r * T;
    if (i < mb) {
#pragma unroll
      for (int j = 0; j < NMAX; ++j)
        if (j < n) Qo[(r0 + i) + (int64_t)j * ldq] = sg[j] * a[r][j];
    }
  }
}

// ---- Householder QR with the compact WY Q (n <= 16) ---------------------
// The leaf QR of the rounding sweeps (512 x 16 blocks) is a latency chain:
// column step c needs the reduction of step c - 1.  Each step here is one
// CTA-wide reduction (all NMAX partial dots of the pivot column at once,
// staged through shared memory: every thread writes its NMAX partials, G
// threads per slot sum them, a G-lane shuffle finishes), two barriers, and
// the pivot scalars recomputed by every thread (bit-identical, no third
// barrier).  Columns stay at fixed registers (runtime column c picked by a
// uniform switch), and the finished columns of the registers ARE the
// reflectors V, so the partials of step c also give V^T v_c for free:
// the WY factor T of H_0 .. H_{k-1} = I - V T V^T is built as the steps go,
// and Q = [I; 0] - V (T V_1^T) is one per-row product at the end instead of
// k more sequential reduction steps.
template <int NMAX>
struct WyScratch {
  double rowc[2][NMAX];  // pivot row of step c (double-buffered by parity)
  double tot[NMAX];      // slot totals of step c
  double tau[NMAX], beta[NMAX];
  double Tm[NMAX][NMAX + 1];  // WY T factor (upper triangular)
  double Vt[NMAX][NMAX + 1];  // rows j < k of V
  double Mm[NMAX][NMAX + 1];  // T V_1^T (or T V_1^T P for the SVD kernel)
  double Rm[NMAX][NMAX + 1];  // R (rows < min(mb, n))
};

// Householder QR of the mb x n block held in a[RPT][NMAX] (row i = t + r NT,
// NT = blockDim.x, a power of two with NT / NMAX <= 32).  Rotating layout:
// at step c the pivot column is register 0, the live trailing columns
// 1 .. n - c - 1, then the zero padding, then the finished reflectors
// V_0 .. V_{c-1} (V_q at NMAX - c + q): after the step the row rotates left
// by one and the new reflector entry enters at the end.  So the loop body is
// one compact block (the fully unrolled variant was instruction-fetch bound)
// and the partials of the pivot column against the V registers are exactly
// the V^T v_c terms of the WY T factor.  NMAX rotations in total, so on exit
// a[r][q] = V(i, q) for q < k.  sc.Rm = R (rows < min(mb, n)), sc.Tm = T,
// sc.Vt = V rows < k, sc.tau / sc.beta; part = NMAX x NT doubles of shared
// scratch.
template <int NMAX, int RPT, int NT>
__device__ void wy_qr(double (&a)[RPT][NMAX], int mb, int n, double *part, WyScratch<NMAX> &sc) {
  constexpr int G = NT / NMAX;  // threads per slot in the reduction
  static_assert(G >= 1 && G <= 32 && (G & (G - 1)) == 0, "slot groups");
  const int t = threadIdx.x;
  const int k = min(mb, n);
  for (int c = 0; c < NMAX; ++c) {
    if (c < k) {
      const int nc = n - c;
      if (t == c) {
#pragma unroll
        for (int u = 0; u < NMAX; ++u) sc.rowc[c & 1][u] = a[0][u];
      }
      double x[RPT];
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int i = t + r * NT;
        x[r] = (i > c && i < mb) ? a[r][0] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < NMAX; ++u) {
        double p = 0.0;
#pragma unroll
        for (int r = 0; r < RPT; ++r) p = fma(x[r], a[r][u], p);
        part[u * NT + t] = p;
      }
      __syncthreads();
      {
        const int u = t / G, g = t - u * G;
        const double *pu = part + u * NT + g;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int j = 0; j < NMAX; j += 4) {
          s0 += pu[(j + 0) * G];
          if (j + 1 < NMAX) s1 += pu[(j + 1) * G];
          if (j + 2 < NMAX) s2 += pu[(j + 2) * G];
          if (j + 3 < NMAX) s3 += pu[(j + 3) * G];
        }
        double s = (s0 + s1) + (s2 + s3);
#pragma unroll
        for (int o = G >> 1; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (g == 0) sc.tot[u] = s;
      }
      __syncthreads();
      const double *rc = sc.rowc[c & 1];
      const double xx = sc.tot[0], alpha = rc[0];
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
      if (t == 0) {
        sc.tau[c] = tau;
        sc.beta[c] = beta;
      }
      // T(0:c, c) = -tau T(0:c, 0:c) (V^T v_c)(0:c), (V^T v_c)(q) = V(c, q) + scal tot(q)
      // with V_q at register NMAX - c + q
      if (t < c) {
        double acc = 0.0;
        for (int q = t; q < c; ++q) {
          const int pq = NMAX - c + q;
          acc = fma(sc.Tm[t][q], fma(scal, sc.tot[pq], rc[pq]), acc);
        }
        sc.Tm[t][c] = -tau * acc;
      } else if (t == c) {
        sc.Tm[c][c] = tau;
      }
      // w(u) = v_c^T a_u for the live columns 1 <= u < n - c
      double w[NMAX];
#pragma unroll
      for (int u = 1; u < NMAX; ++u) w[u] = u < nc ? fma(scal, sc.tot[u], rc[u]) : 0.0;
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int i = t + r * NT;
        if (i > c && i < mb) {
          const double v = scal * a[r][0];
          const double tv = tau * v;
#pragma unroll
          for (int u = 1; u < NMAX; ++u) a[r][u] = fma(-w[u], tv, a[r][u]);
          a[r][0] = v;
        } else if (i == c) {
#pragma unroll
          for (int u = 1; u < NMAX; ++u) a[r][u] = fma(-tau, w[u], a[r][u]);
          sc.Rm[c][c] = beta;
          a[r][0] = 1.0;
        } else {
          if (i < c) sc.Rm[i][c] = a[r][0];  // R(i, c), final since step i
          a[r][0] = 0.0;
        }
      }
    } else if (c == k) {
      // wide block (mb < n): the trailing columns k .. n-1 sit at 0 .. n-k-1
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int i = t + r * NT;
        if (i < k) {
#pragma unroll
          for (int u = 0; u < NMAX; ++u)
            if (u < n - k) sc.Rm[i][k + u] = a[r][u];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const double v0 = a[r][0];
#pragma unroll
      for (int u = 0; u + 1 < NMAX; ++u) a[r][u] = a[r][u + 1];
      a[r][NMAX - 1] = v0;
    }
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = t + r * NT;
    if (i < k) {
#pragma unroll
      for (int u = 0; u < NMAX; ++u)
        if (u < k) sc.Vt[i][u] = a[r][u];
    }
  }
  __syncthreads();
}

// Columns [J0, J0 + NC) of Q = Z0 - V M for this thread's rows: q(r, jj) for
// column J0 + jj, Z0 = [Ztop; 0] (Ztop k x ncol, identity when ztop is null).
template <int NMAX, int RPT, int J0, int NC>
__device__ __forceinline__ void wy_rows(const double (&a)[RPT][NMAX], int k, int ncol,
                                        const double (*Mm)[NMAX + 1], const double (*ztop)[NMAX + 1],
                                        double (&q)[RPT][NC]) {
  const int t = threadIdx.x, T = blockDim.x;
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = t + r * T;
#pragma unroll
    for (int jj = 0; jj < NC; ++jj) {
      const int j = J0 + jj;
      q[r][jj] = (i < k && j < ncol) ? (ztop ? ztop[i][j] : (i == j ? 1.0 : 0.0)) : 0.0;
    }
  }
#pragma unroll
  for (int a2 = 0; a2 < NMAX; ++a2) {
    if (a2 >= k) break;
#pragma unroll
    for (int jj = 0; jj < NC; ++jj) {
      const double mj = J0 + jj < ncol ? Mm[a2][J0 + jj] : 0.0;
#pragma unroll
      for (int r = 0; r < RPT; ++r) q[r][jj] = fma(-a[r][a2], mj, q[r][jj]);
    }
  }
}

// Q rows of this thread to Qo (column j scaled by sg(j)), NC columns at a time.
template <int NMAX, int RPT, int J0>
__device__ __forceinline__ void wy_store(const double (&a)[RPT][NMAX], int k, int n, int mb,
                                         const double (*Mm)[NMAX + 1],
                                         const double (*ztop)[NMAX + 1], const double *sg,
                                         double *__restrict__ Qo, int64_t ldq, int64_t r0) {
  constexpr int NC = NMAX < 8 ? NMAX : 8;
  if constexpr (J0 < NMAX) {
    double q[RPT][NC];
    wy_rows<NMAX, RPT, J0, NC>(a, k, ztop ? n : k, Mm, ztop, q);
    const int t = threadIdx.x, T = blockDim.x;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = t + r * T;
      if (i < mb) {
#pragma unroll
        for (int jj = 0; jj < NC; ++jj)
          if (J0 + jj < n) Qo[(r0 + i) + (int64_t)(J0 + jj) * ldq] = sg[J0 + jj] * q[r][jj];
      }
    }
    wy_store<NMAX, RPT, J0 + NC>(a, k, n, mb, Mm, ztop, sg, Qo, ldq, r0);
  }
}

// TSQR level for n <= 16 with the WY Q (same outputs as k_tsqr_level).
template <int NMAX, int RPT>
__global__ void __launch_bounds__(LEAF_MAX / RPT) k_tsqr_wy(
    int64_t M, int n, const double *__restrict__ A, int64_t lda, int trans, double *__restrict__ Rs,
    int64_t ldr, double *__restrict__ Qo, int64_t ldq, int root, int *__restrict__ status) {
  extern __shared__ double part[];  // NMAX x blockDim
  __shared__ WyScratch<NMAX> sc;
  const int T = blockDim.x, t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * T * RPT;
  const int mb = (int)min((int64_t)T * RPT, M - r0);
  const int k = min(mb, n);
  double a[RPT][NMAX];
  if (!load_rows<NMAX, RPT>(a, mb, n, A, lda, trans, r0)) {
    if (t == 0) atomicOr(status, 1);
    return;
  }
  wy_qr<NMAX, RPT, LEAF_MAX / RPT>(a, mb, n, part, sc);
  // M = T V_1^T:  M(q, j) = sum_{b = q .. j} T(q, b) V(j, b)   (V(j, j) = 1)
  for (int e = t; e < k * k; e += T) {
    const int q = e / k, j = e - q * k;
    double acc = 0.0;
    for (int b = q; b <= j; ++b) acc = fma(sc.Tm[q][b], sc.Vt[j][b], acc);
    sc.Mm[q][j] = acc;
  }
  if (Rs && t < n) {  // row t of R_b (sign-fixed at the root)
    const double sg = (root && t < k && sc.beta[t] < 0.0) ? -1.0 : 1.0;
    const int64_t rb = (int64_t)blockIdx.x * n + t;
    for (int j = 0; j < n; ++j)
      Rs[rb + (int64_t)j * ldr] = (t <= j && t < mb) ? sg * sc.Rm[t][j] : 0.0;
  }
  if (t < NMAX) sc.tot[t] = t < k ? ((root && sc.beta[t] < 0.0) ? -1.0 : 1.0) : 0.0;  // column signs
  __syncthreads();
  wy_store<NMAX, RPT, 0>(a, k, n, mb, sc.Mm, nullptr, sc.tot, Qo, ldq, r0);
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

// The same stage for n <= 16 by one warp out of registers (warp_jacobi_cols).
template <int NM>
__global__ void __launch_bounds__(32) k_jacobi_warp(int n, const double *__restrict__ R, int64_t ldr,
                                                    double *__restrict__ Yo, double *__restrict__ Po,
                                                    double *__restrict__ norms, int max_sweeps,
                                                    int *__restrict__ status) {
  __shared__ double X[NM * NM], P[NM * NM];
  const int lane = threadIdx.x;
  double f = 0.0;
  for (int e = lane; e < n * n; e += 32) {
    const int j = e / n, i = e - j * n;  // X(i, j) = R(j, i)
    const double v = j <= i ? R[j + (int64_t)i * ldr] : 0.0;
    X[e] = v;
    P[e] = i == j ? 1.0 : 0.0;
    f += v * v;
  }
  const double fro2 = warp_sum(f);
  __syncwarp();
  const double tol = kEps * sqrt((double)n);
  const double floor = 0.01 * kEps * kEps * (double)n * fro2;
  const int sweeps = warp_jacobi_cols<NM>(X, n, P, n, n, tol, floor, max_sweeps);
  if (lane == 0) {
    status[1] = sweeps;
    if (sweeps < 0) atomicOr(status, 2);
  }
  if (lane < n) {
    double s2 = 0.0;
    for (int i = 0; i < n; ++i) s2 = fma(X[i + lane * n], X[i + lane * n], s2);
    norms[lane] = sqrt(s2);
  }
  for (int e = lane; e < n * n; e += 32) {
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
  FTT_CUDA(cudaFuncSetAttribute(k_tsqr_level_m<8, 1>, a, cap));
  FTT_CUDA(cudaFuncSetAttribute(k_tsqr_level_m<8, 2>, a, cap));
  FTT_CUDA(cudaFuncSetAttribute(k_tsqr_level_m<8, 4>, a, cap));
  FTT_CUDA(cudaFuncSetAttribute(k_tsqr_level_m<16, 1>, a, cap));
  FTT_CUDA(cudaFuncSetAttribute(k_tsqr_level_m<16, 2>, a, cap));
  FTT_CUDA(cudaFuncSetAttribute(k_tsqr_level_m<16, 4>, a, cap));
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
  // n <= 16: rpt rows per thread
  const int rpt = LEAF_RPT;  // (4 rows per thread measured slower: DESIGN 4e)
  const unsigned ntm = (unsigned)(leaf / rpt);  // k_tsqr_wy's compile-time thread count
  switch (nmax_for(n)) {
    case 8:
      if (rpt == 4)
        k_tsqr_wy<8, 4><<<grid, ntm, 8 * 8 * ntm, ctx->stream>>>(M, n, A, lda, trans, Rs, ldr, Qo,
                                                                 ldq, root, status);
      else
        k_tsqr_wy<8, 2><<<grid, ntm, 8 * 8 * ntm, ctx->stream>>>(M, n, A, lda, trans, Rs, ldr, Qo,
                                                                 ldq, root, status);
      break;
    case 16:
      if (rpt == 4)
        k_tsqr_wy<16, 4><<<grid, ntm, 8 * 16 * ntm, ctx->stream>>>(M, n, A, lda, trans, Rs, ldr, Qo,
                                                                   ldq, root, status);
      else
        k_tsqr_wy<16, 2><<<grid, ntm, 8 * 16 * ntm, ctx->stream>>>(M, n, A, lda, trans, Rs, ldr, Qo,
                                                                   ldq, root, status);
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

// SVD of a short tall block (m x n, n <= 16, m <= SV_NT * RPT) in one CTA:
// the WY Householder QR of the TSQR leaves (wy_qr), one-sided Jacobi on
// X = R^T by warp 0 out of registers (warp_jacobi_cols; the rows of R are
// the better-conditioned Jacobi operand) while the other warps form
// M = T V_1^T, then U = Q [P; 0] = [P; 0] - V (M P) per row.  Outputs as
// tsqr_svd: Uo = Q P (m x n, ld m), Yo = X P (n x n, column norms sigma_j),
// so A_tall = U Sigma (Yo / sigma)^T.  For the inner factor B of the
// low-rank path (512 x 16 on config 5) this is one launch instead of a TSQR
// tree, a Jacobi launch and the Q expansion.
constexpr int SV_NT = 256;
template <int NMAX, int RPT>
__global__ void __launch_bounds__(SV_NT) k_svd_wy(int m, int n, const double *__restrict__ A,
                                                  int64_t lda, int trans, double *__restrict__ Uo,
                                                  double *__restrict__ Yo,
                                                  double *__restrict__ norms, int max_sweeps,
                                                  int *__restrict__ status,
                                                  const double *__restrict__ extra_src,
                                                  double *__restrict__ extra_dst) {
  extern __shared__ double part[];  // NMAX x SV_NT
  __shared__ WyScratch<NMAX> sc;
  __shared__ double X[NMAX * NMAX], P[NMAX * NMAX];
  __shared__ double red[SV_NT / 32];
  __shared__ int s_sweeps;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double a[RPT][NMAX];
  if (t == 0 && extra_src) *extra_dst = *extra_src;
  if (!load_rows<NMAX, RPT>(a, m, n, A, lda, trans, 0)) {
    if (t == 0) {
      status[0] = 1;
      status[1] = 0;
    }
    return;
  }
  double f = 0.0;
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int u = 0; u < NMAX; ++u) f = fma(a[r][u], a[r][u], f);
  const double fro2 = cta_sum(f, red);
  wy_qr<NMAX, RPT, SV_NT>(a, m, n, part, sc);
  for (int e = t; e < n * n; e += SV_NT) {  // X = R^T, P = I
    const int b = e / n, i = e - b * n;
    X[e] = b <= i ? sc.Rm[b][i] : 0.0;
    P[e] = i == b ? 1.0 : 0.0;
  }
  __syncthreads();
  if (warp == 0) {
    const double tol = kEps * sqrt((double)n);
    const double floor = 0.01 * kEps * kEps * (double)m * fro2;
    const int sw = warp_jacobi_cols<NMAX>(X, n, P, n, n, tol, floor, max_sweeps);
    if (lane == 0) s_sweeps = sw;
  } else {
    // M = T V_1^T:  M(q, j) = sum_{b = q .. j} T(q, b) V(j, b)   (V(j, j) = 1)
    for (int e = t - 32; e < n * n; e += SV_NT - 32) {
      const int q = e / n, j = e - q * n;
      double acc = 0.0;
      for (int b = q; b <= j; ++b) acc = fma(sc.Tm[q][b], sc.Vt[j][b], acc);
      sc.Mm[q][j] = acc;
    }
  }
  __syncthreads();
  // (M P) into Rm, P row-major into Vt (both free now)
  for (int e = t; e < n * n; e += SV_NT) {
    const int q = e / n, j = e - q * n;
    double acc = 0.0;
    for (int b = 0; b < n; ++b) acc = fma(sc.Mm[q][b], P[b + j * n], acc);
    sc.Rm[q][j] = acc;
    sc.Vt[q][j] = P[q + j * n];
  }
  if (t < NMAX) sc.tot[t] = 1.0;  // no column signs
  __syncthreads();
  wy_store<NMAX, RPT, 0>(a, n, n, m, sc.Rm, sc.Vt, sc.tot, Uo, m, 0);
  if (t == 0) {
    status[0] = s_sweeps < 0 ? 2 : 0;
    status[1] = s_sweeps;
  }
  if (t < n) {
    double s2 = 0.0;
    for (int i = 0; i < n; ++i) s2 = fma(X[i + t * n], X[i + t * n], s2);
    norms[t] = sqrt(s2);
  }
  for (int e = t; e < n * n; e += SV_NT) Yo[e] = X[e];
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
             const double *extra_dev, double *extra_host, int extra_n) {
  const int n = (int)n64;
  FTT_CHECK(set_attrs());
  double *dev = nullptr;
  // status (2 ints) | extra | norms n | extras 1..3, pad | R n x n | P n x n
  // (R keeps the 16-byte alignment it had without the extras)
  FTT_CHECK(owned_alloc(ctx, (void **)&dev, 8 * (size_t)(2 + n + 4 + 2 * (size_t)n * n)));
  int *status = reinterpret_cast<int *>(dev);
  double *norms = dev + 2;
  double *R = norms + n + 4;
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
  if (n <= 8)
    k_jacobi_warp<8><<<1, 32, 0, ctx->stream>>>(n, R, n, Y, P, norms, max_sweeps, status);
  else if (n <= 16)
    k_jacobi_warp<16><<<1, 32, 0, ctx->stream>>>(n, R, n, Y, P, norms, max_sweeps, status);
  else
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
  const int xn = extra_dev ? std::max(1, std::min(extra_n, 4)) : 1;
  if (extra_dev) {
    FTT_CUDA(cudaMemcpyAsync(dev + 1, extra_dev, sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    if (xn > 1)
      FTT_CUDA(cudaMemcpyAsync(dev + 2 + n, extra_dev + 1, sizeof(double) * (xn - 1),
                               cudaMemcpyDeviceToDevice, ctx->stream));
  }
  std::vector<double> h(n + 2 + 3);
  FTT_CHECK(copy_to_host(ctx, h.data(), dev, 8 * (size_t)(n + 1 + xn)));
  if (extra_dev && extra_host) {
    extra_host[0] = h[1];
    for (int x = 1; x < xn; ++x) extra_host[x] = h[n + 1 + x];
  }
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
  return !off && n >= 1 && n <= 16 && m >= n && m <= 4 * SV_NT;
}

// SVD of the short tall A_tall (m x n) in one launch (k_svd_wy): U = Q P
// (m x n, ld m), Yt = R^T P (n x n, ld n), norms_host[j] = ||Yt_j||
// (unsorted) -- the outputs of tsqr_svd.
int direct_small_svd(ftt_ctx *ctx, int64_t m, int64_t n, const double *A, int64_t lda, int trans,
                     double *U, double *Yt, double *norms_host, int *sweeps,
                     const double *extra_dev, double *extra_host, int extra_n) {
  double *dev = nullptr;  // status (2 ints) | extra | norms n | extras 1..3
  FTT_CHECK(owned_alloc(ctx, (void **)&dev, 8 * (size_t)(2 + n + 3)));
  int *status = reinterpret_cast<int *>(dev);
  const int max_sweeps = 60;
  const size_t smem = 8 * (size_t)(n <= 8 ? 8 : 16) * SV_NT;
#define FTT_SVD_WY(NM, R)                                                                      \
  k_svd_wy<NM, R><<<1, SV_NT, smem, ctx->stream>>>((int)m, (int)n, A, lda, trans, U, Yt, dev + 2, \
                                                   max_sweeps, status, extra_dev, dev + 1)
  if (n <= 8) {
    if (m <= 2 * SV_NT) FTT_SVD_WY(8, 2);
    else FTT_SVD_WY(8, 4);
  } else {
    if (m <= 2 * SV_NT) FTT_SVD_WY(16, 2);
    else FTT_SVD_WY(16, 4);
  }
#undef FTT_SVD_WY
  FTT_LAUNCHED(ctx);
  const int xn = extra_dev ? std::max(1, std::min(extra_n, 4)) : 1;
  if (extra_dev && xn > 1)
    FTT_CUDA(cudaMemcpyAsync(dev + 2 + n, extra_dev + 1, sizeof(double) * (xn - 1),
                             cudaMemcpyDeviceToDevice, ctx->stream));
  std::vector<double> h(n + 2 + 3);
  FTT_CHECK(copy_to_host(ctx, h.data(), dev, 8 * (size_t)(n + 1 + xn)));
  if (extra_dev && extra_host) {
    extra_host[0] = h[1];
    for (int x = 1; x < xn; ++x) extra_host[x] = h[n + 1 + x];
  }
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
