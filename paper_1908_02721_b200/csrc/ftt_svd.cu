// Thin fp64 SVD for the truncation steps of the rounding sweeps
// (svd_truncate_delta / svd_truncate_rank, linalg.py:75-125, whose
// _full_svd is LAPACK gesdd, linalg.py:48-53).
//
// Backward-stable, no Gram-matrix shortcut:
//   A (m_A x n_A, m_A >= n_A; the transpose is taken for wide inputs)
//     = Q R                      blocked Householder QR (ftt_qr.cu)
//   X = R^T,  X P = Y            one-sided block Jacobi: columns of X are
//                                orthogonalised by right rotations P
//   sigma_j = ||Y_j||,  A = (Q P) diag(sigma) (Y diag(1/sigma))^T
// Block Jacobi: columns in blocks of 16; a round-robin tournament pairs the
// blocks so every step processes nblk/2 disjoint 32-column pairs, one CTA
// each.  A CTA forms the 32x32 Gram of its pair from the CURRENT columns
// (fresh dot products, so each entry is accurate relative to its own column
// norms), diagonalises it with cyclic two-sided Jacobi in shared memory
// (Rutishauser rotation, relative threshold tol*sqrt(g_pp g_qq)), and applies
// the accumulated 32x32 rotation to the pair's columns of X and P.  A sweep
// with no rotation anywhere ends the iteration.
#include <algorithm>
#include <atomic>
#include <numeric>
#include <vector>

#include <cooperative_groups.h>

#include "ftt_dense.cuh"
#include "ftt_small.cuh"

namespace cg = cooperative_groups;

namespace ftt {

int launch_identity(ftt_ctx *ctx, int64_t m, int64_t k, double *Z, int64_t ldz);

struct SvdState {
  int64_t m = 0, n = 0;    // caller's shape
  int64_t mA = 0, nA = 0;  // tall orientation
  bool transposed = false;
  double *Af = nullptr;    // factored A (mA x nA)
  double *tau = nullptr;
  double *Tb = nullptr;
  double *Y = nullptr;     // nA x nA (X after Jacobi)
  double *P = nullptr;     // nA x nA accumulated rotations
  double *B = nullptr;     // nA x nA: QR of R^T (preconditioning), reflectors
  double *tau2 = nullptr;
  double *Tb2 = nullptr;
  std::vector<double> sigma;  // sorted descending
  std::vector<int64_t> perm;  // sorted position -> column of Y
  int sweeps = 0;
  bool precond = false;  // Jacobi ran on R2^T (QR of R^T) instead of R^T
  // Jacobi ran on R2^T with R Pi = Q2 R2 (pivoted QR of R: A Pi = (Q Q2) R2);
  // B holds Q2's reflectors and R2, piv the pivoting (device ints)
  bool pivoted = false;
  int *piv = nullptr;
  bool direct = false;   // Jacobi ran on A_tall itself (Y aliases Af)
  bool small = false;    // narrow path (ftt_small.cu): Af holds U = Q P, Y = R^T P
  // low-rank path (ftt_svd_lowrank_f64): A_tall ~= Qk Bk with a certified
  // residual; the SVD of the small Bk lives in `inner`
  bool lowrank = false;
  double *Qk = nullptr;  // mA x k orthonormal range basis
  double *Bk = nullptr;  // k x nA
  SvdState *inner = nullptr;
};

void svd_state_free(ftt_ctx *ctx);
void svd_state_release(ftt_ctx *ctx, SvdState *s);

namespace {

constexpr int JB = 16;
constexpr int JP = 2 * JB;  // 32 columns per pair
constexpr int JT = 256;
constexpr int CH = 64;      // rows per staged chunk
// Inner two-sided sweeps on the pair's Gram before the next fresh
// recompute.  They only pick rotations (convergence is decided on fresh
// Grams), and each costs 31 rounds x 3 CTA barriers: measured on config 4's
// 2064 x 766 operand, 1 inner sweep = 23 outer sweeps / 97 ms, 3 = 21 / 153 ms.
__device__ int g_max_inner = 1;  // inner two-sided sweeps per block pair (up to 3 supported)
int g_last_csize = 1;             // debug print only

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Column streams of a pair go through an NSTAGE-deep cp.async pipeline
// (4 stages at 2 CTAs per SM by default, 3 stages at 3 CTAs per SM): a
// stage is one 64-row chunk of the pair's 32 columns stored column-major
// with a 68-double column stride (16-byte aligned; the DMMA fragment reads
// of both the Gram and the rotation hit every bank pair at most twice, the
// minimum for 32 doubles).  Deep pipelining is what the pair loop needs:
// one CTA per SM streams ~1.3 MB per column pass, and a single chunk in
// flight left it latency bound at ~1.3 TB/s over the GPU.
constexpr int CHS = CH + 4;
constexpr int STAGE_ELEMS = JP * CHS;
constexpr size_t jac_dyn_bytes(int ns) { return sizeof(double) * ns * STAGE_ELEMS; }
constexpr int JAC_GP_OFF = (JT / 32) * 10 * 64;  // Gram of this CTA, after the warp partials
static_assert(3 * STAGE_ELEMS >= JAC_GP_OFF + JP * JP, "Gram partials fit the stages");

__device__ __forceinline__ void cp_async16(double *smem, const double *gmem, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async8(double *smem, const double *gmem, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Issue the copies of rows [r0, r0 + CH) of the pair's columns into one
// stage (zero-filled past `rows` and for padding columns).
__device__ __forceinline__ void chunk_issue(double *stage, const double *__restrict__ M, int64_t r0,
                                            int64_t rows, int64_t ld, const int *col, int tid,
                                            bool vec16) {
  if (vec16) {
#pragma unroll
    for (int q = 0; q < CH * JP / 2 / JT; ++q) {
      const int e = q * JT + tid;
      const int c = e >> 5, seg = e & 31;
      const int64_t row = r0 + 2 * seg;
      const int cc = col[c];
      const int bytes = (cc < 0 || row >= rows) ? 0 : (row + 1 < rows ? 16 : 8);
      cp_async16(stage + c * CHS + 2 * seg, bytes ? M + row + (int64_t)cc * ld : M, bytes);
    }
  } else {
#pragma unroll
    for (int q = 0; q < CH * JP / JT; ++q) {
      const int e = q * JT + tid;
      const int c = e >> 6, r = e & 63;
      const int64_t row = r0 + r;
      const int cc = col[c];
      const int bytes = (cc < 0 || row >= rows) ? 0 : 8;
      cp_async8(stage + c * CHS + r, bytes ? M + row + (int64_t)cc * ld : M, bytes);
    }
  }
}

__device__ __forceinline__ void pair_of(int nblk, int step, int c, int *a, int *b) {
  // circle method, team nblk-1 fixed
  const int L = nblk - 1;
  if (c == 0) {
    *a = step;
    *b = L;
  } else {
    *a = (step + c) % L;
    *b = (step - c + L) % L;
  }
}

// One Jacobi step: CTA c handles block pair pair_of(nblk, step, c).
// Convergence is decided on the FRESH Gram only (entries from the current
// columns): pair (i, j) needs work iff both columns are above the noise
// floor (|x|^2 > floor) and |g_ij| > tol sqrt(g_ii g_jj).  The inner
// two-sided sweeps (at most 3) use Rutishauser's diagonal update
// g_pp -= t g_pq, g_qq += t g_pq; entries derived there are only used to
// pick the next rotations, never to declare convergence, so rounding in
// them (after cancellation between near-parallel columns) cannot stall the
// iteration -- the next step recomputes them from the rotated columns.
struct JacSmem {
  double G[JP][JP + 1];
  double Z[JP][JP + 1];
  double rc[16], rs[16], rt[16], rpp[16], rqq[16], rpq[16];
  int col[JP];
  int s_round_any;
  unsigned char tp[JP - 1][16], tq[JP - 1][16];  // inner round-robin pairing table
};

// Exact work skipping (track != nullptr): last_mod[b] = global step at which
// block b was last rotated, last_ok[a*nblk+b] = global step at which pair
// (a, b) last passed the fresh convergence test.  If neither block changed
// since that test, recomputing its Gram would reproduce the same data and
// the same "no rotation" outcome, so the pair is skipped without reading X.
struct JacTrack {
  int *last_mod;
  int *last_ok;
  int t;  // global step index (sweep * (nblk - 1) + step)
};

// n columns; X is mX x n (ld ldx), P is n x n (ld ldp).  NSTAGE-deep
// column pipeline.
template <int NSTAGE>
__device__ void jacobi_pair(int64_t n, int64_t mX, double *__restrict__ X, int64_t ldx,
                            double *__restrict__ P, int64_t ldp,
                            int nblk, int step, int pc, double tol, double floor,
                            unsigned long long *__restrict__ rotated, JacSmem &sm,
                            double *__restrict__ stages, int crank, int csize,
                            const JacTrack *track = nullptr) {
  auto &G = sm.G;
  auto &Z = sm.Z;
  auto &rc = sm.rc;
  auto &rs = sm.rs;
  auto &rt = sm.rt;
  auto &rpp = sm.rpp;
  auto &rqq = sm.rqq;
  auto &rpq = sm.rpq;
  auto &col = sm.col;
  const int tid = threadIdx.x;
  __syncthreads();  // the previous pair of this CTA is done with sm
  int ba, bb;
  pair_of(nblk, step, pc, &ba, &bb);
  const int pidx = min(ba, bb) * nblk + max(ba, bb);
  if (track) {
    int skip = 0;
    if (tid == 0) {
      const int ok = __ldcg(track->last_ok + pidx);
      skip = ok > __ldcg(track->last_mod + ba) && ok > __ldcg(track->last_mod + bb);
    }
    if (__syncthreads_or(skip)) return;
  }
  for (int e = tid; e < (JP - 1) * 16; e += JT) {
    int p, q;
    pair_of(JP, e / 16, e % 16, &p, &q);
    sm.tp[e / 16][e % 16] = (unsigned char)p;
    sm.tq[e / 16][e % 16] = (unsigned char)q;
  }
  if (tid < JP) {
    int blk = tid < JB ? ba : bb;
    int cidx = blk * JB + (tid % JB);
    col[tid] = cidx < n ? cidx : -1;
  }
  __syncthreads();
  // ---- Gram of the pair's current columns on the DMMA pipe.  Only the 10
  // upper 8x8 tiles are formed; warp w takes k-steps w and w + 8 of every
  // 64-row chunk for all 10 tiles (4 fragment loads feed 10 MMAs), and the
  // eight partial Grams are summed in fixed warp order afterwards.
  const int lane = tid & 31, warp = tid >> 5;
  const int gi = tid >> 3;          // convergence test: row of G
  const int gj = (tid & 7) * 4;     //   and 4 consecutive columns
  const bool vx16 = ((reinterpret_cast<uintptr_t>(X) & 15) == 0) && !(ldx & 1);
  // row slice of this CTA within its cluster (whole 64-row chunks)
  auto slice = [&](int64_t rows, int64_t *c_lo, int64_t *c_hi) {
    const int64_t nch = (rows + CH - 1) / CH, per = (nch + csize - 1) / csize;
    *c_lo = min(nch, per * crank);
    *c_hi = min(nch, per * (crank + 1));
  };
  int64_t gx0, gx1;
  slice(mX, &gx0, &gx1);
  const int64_t nchX = gx1 - gx0;
  const double *Xs = X + gx0 * CH;  // rows of the slice start here
  const int64_t mXs = min(mX - gx0 * CH, nchX * CH);
  {
    double gacc[10][2];
#pragma unroll
    for (int t = 0; t < 10; ++t) gacc[t][0] = gacc[t][1] = 0.0;
#pragma unroll
    for (int c = 0; c < NSTAGE - 1; ++c) {
      if (c < nchX) chunk_issue(stages + c * STAGE_ELEMS, Xs, c * CH, mXs, ldx, col, tid, vx16);
      cp_async_commit();
    }
    for (int64_t c = 0; c < nchX; ++c) {
      cp_async_wait<NSTAGE - 2>();
      __syncthreads();
      if (c + NSTAGE - 1 < nchX)
        chunk_issue(stages + ((c + NSTAGE - 1) % NSTAGE) * STAGE_ELEMS, Xs, (c + NSTAGE - 1) * CH,
                    mXs, ldx, col, tid, vx16);
      cp_async_commit();
      const double *Sb = stages + (c % NSTAGE) * STAGE_ELEMS;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int k = (warp + 8 * kk) * 4 + (lane & 3);
        double f[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) f[t] = Sb[(t * 8 + (lane >> 2)) * CHS + k];
        int idx = 0;
#pragma unroll
        for (int ti = 0; ti < 4; ++ti)
#pragma unroll
          for (int tj = ti; tj < 4; ++tj, ++idx) dmma(gacc[idx][0], gacc[idx][1], f[ti], f[tj]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    double *part = stages;  // [warp][tile][64]
#pragma unroll
    for (int t = 0; t < 10; ++t) {
      part[(warp * 10 + t) * 64 + (lane >> 2) * 8 + 2 * (lane & 3)] = gacc[t][0];
      part[(warp * 10 + t) * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = gacc[t][1];
    }
    __syncthreads();
    // this CTA's Gram (both triangles) -> Gp (in the stages, past the
    // partials); with a cluster the members' Gp are summed in rank order, so
    // every member holds the bitwise same G
    double *Gp = stages + JAC_GP_OFF;
    for (int e = tid; e < 640; e += JT) {
      const int t = e >> 6, w = e & 63;
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < JT / 32; ++q) v += part[(q * 10 + t) * 64 + w];
      const int ti = t < 4 ? 0 : t < 7 ? 1 : t < 9 ? 2 : 3;
      const int tj = ti + t - (ti == 0 ? 0 : ti == 1 ? 4 : ti == 2 ? 7 : 9);
      const int i = ti * 8 + (w >> 3), j = tj * 8 + (w & 7);
      if (i <= j) {
        Gp[i * JP + j] = v;
        Gp[j * JP + i] = v;
      }
    }
    if (csize > 1) {
      cg::cluster_group cl = cg::this_cluster();
      cl.sync();
      for (int e = tid; e < JP * JP; e += JT) {
        double v = 0.0;
        for (int r = 0; r < csize; ++r) v += cl.map_shared_rank(Gp, r)[e];
        G[e / JP][e % JP] = v;
      }
      cl.sync();  // members' Gp no longer read
    } else {
      __syncthreads();
      for (int e = tid; e < JP * JP; e += JT) G[e / JP][e % JP] = Gp[e];
    }
  }
  for (int e = tid; e < JP * JP; e += JT) Z[e / JP][e % JP] = (e / JP == e % JP) ? 1.0 : 0.0;
  __syncthreads();
  // ---- fresh convergence test
  int need = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int j = gj + q;
    if (j > gi) {
      double dii = G[gi][gi], djj = G[j][j], gij = G[gi][j];
      if (dii > floor && djj > floor && fabs(gij) > tol * sqrt(dii * djj)) need = 1;
    }
  }
  if (!__syncthreads_or(need)) {
    if (track && tid == 0 && crank == 0) track->last_ok[pidx] = track->t;
    return;
  }
  if (track && tid == 0 && crank == 0) {
    track->last_mod[ba] = track->t;
    track->last_mod[bb] = track->t;
  }
  // ---- cyclic two-sided Jacobi on G (parallel: 16 disjoint pairs per round)
  const int max_inner = g_max_inner;
  for (int sw = 0; sw < max_inner; ++sw) {
    int sweep_any = 0;
    for (int round = 0; round < JP - 1; ++round) {
      int flag = 0;
      if (tid < 16) {
        const int p = sm.tp[round][tid], q = sm.tq[round][tid];
        double gpp = G[p][p], gqq = G[q][q], gpq = G[p][q];
        double c = 1.0, s = 0.0, t = 0.0;
        if (gpp > floor && gqq > floor && fabs(gpq) > tol * sqrt(gpp * gqq)) {
          double zeta = (gqq - gpp) / (2.0 * gpq);
          t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          c = 1.0 / sqrt(1.0 + t * t);
          s = c * t;
          flag = 1;
        }
        rc[tid] = c;
        rs[tid] = s;
        rt[tid] = t;
        rpp[tid] = gpp;
        rqq[tid] = gqq;
        rpq[tid] = gpq;
      }
      if (!__syncthreads_or(flag)) continue;  // barrier 1 (uniform)
      sweep_any = 1;
      // G <- J^T G J in one phase: thread (bi, bj) owns the 2x2 block of
      // pairs bi x bj (disjoint, so no read/write overlap); the pair's own
      // diagonal block exactly (Rutishauser).  Z <- Z J: 2 entries each.
      {
        static_assert(JT == 256, "one thread per 2x2 block of the 16 x 16 pairs");
        const int bi = tid >> 4, bj = tid & 15;
        const int p1 = sm.tp[round][bi], q1 = sm.tq[round][bi];
        const double c1 = rc[bi], s1 = rs[bi];
        if (bi == bj) {
          if (s1 != 0.0) {
            G[p1][p1] = rpp[bi] - rt[bi] * rpq[bi];
            G[q1][q1] = rqq[bi] + rt[bi] * rpq[bi];
            G[p1][q1] = 0.0;
            G[q1][p1] = 0.0;
          }
        } else {
          const int p2 = sm.tp[round][bj], q2 = sm.tq[round][bj];
          const double c2 = rc[bj], s2 = rs[bj];
          if (s1 != 0.0 || s2 != 0.0) {
            const double g11 = G[p1][p2], g12 = G[p1][q2], g21 = G[q1][p2], g22 = G[q1][q2];
            const double a11 = c2 * g11 - s2 * g12, a12 = s2 * g11 + c2 * g12;
            const double a21 = c2 * g21 - s2 * g22, a22 = s2 * g21 + c2 * g22;
            G[p1][p2] = c1 * a11 - s1 * a21;
            G[q1][p2] = s1 * a11 + c1 * a21;
            G[p1][q2] = c1 * a12 - s1 * a22;
            G[q1][q2] = s1 * a12 + c1 * a22;
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = tid + h * JT;
          const int pr = e >> 5, r = e & 31;
          const double c = rc[pr], sn = rs[pr];
          if (sn != 0.0) {
            const int p = sm.tp[round][pr], q = sm.tq[round][pr];
            const double zp = Z[r][p], zq = Z[r][q];
            Z[r][p] = c * zp - sn * zq;
            Z[r][q] = sn * zp + c * zq;
          }
        }
      }
      __syncthreads();  // barrier 2
    }
    if (!sweep_any) break;
  }
  __syncthreads();
  // ---- re-orthogonalise Z (one Newton-Schulz step, Z <- 1.5 Z - 0.5 Z Z^T Z):
  // Z carries up to 2*31 rotations per column; without this its 1e-15-level
  // loss of orthogonality compounds over hundreds of block steps into the
  // singular values (1e-13 relative observed); with it P stays orthogonal
  // to ~1e-15 and sigma matches LAPACK to ~2e-15 relative.
  for (int e = tid; e < JP * JP; e += JT) {  // W = Z^T Z into G
    int i = e / JP, j = e % JP;
    double v = 0.0;
#pragma unroll 8
    for (int r = 0; r < JP; ++r) v += Z[r][i] * Z[r][j];
    G[i][j] = v;
  }
  __syncthreads();
  for (int e = tid; e < JP * JP; e += JT) {  // S = 1.5 Z - 0.5 Z W
    int i = e / JP, j = e % JP;
    double v = 0.0;
#pragma unroll 8
    for (int r = 0; r < JP; ++r) v += Z[i][r] * G[r][j];
    stages[e] = 1.5 * Z[i][j] - 0.5 * v;
  }
  __syncthreads();
  for (int e = tid; e < JP * JP; e += JT) Z[e / JP][e % JP] = stages[e];
  __syncthreads();
  if (tid == 0 && crank == 0) atomicAdd(rotated, 1ull);
  // ---- apply Z to the pair's columns of X and P on the DMMA pipe: warp w
  // owns rows 8w..8w+7 of every 64-row chunk (4 output tiles), the Z
  // fragments stay in registers for the whole pair
  double bz[4][8];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) bz[j][ks] = Z[ks * 4 + (lane & 3)][j * 8 + (lane >> 2)];
  for (int mat = 0; mat < 2; ++mat) {
    double *M = mat == 0 ? X : P;
    const int64_t ld = mat == 0 ? ldx : ldp;
    const bool v16 = ((reinterpret_cast<uintptr_t>(M) & 15) == 0) && !(ld & 1);
    int64_t c0, c1;
    slice(mat == 0 ? mX : n, &c0, &c1);
    M += c0 * CH;
    const int64_t rows = min((mat == 0 ? mX : n) - c0 * CH, (c1 - c0) * CH);
    const int64_t nch = c1 - c0;
    __syncthreads();  // stages free (Newton-Schulz scratch / previous matrix)
#pragma unroll
    for (int c = 0; c < NSTAGE - 1; ++c) {
      if (c < nch) chunk_issue(stages + c * STAGE_ELEMS, M, c * CH, rows, ld, col, tid, v16);
      cp_async_commit();
    }
    for (int64_t c = 0; c < nch; ++c) {
      cp_async_wait<NSTAGE - 2>();
      __syncthreads();
      if (c + NSTAGE - 1 < nch)
        chunk_issue(stages + ((c + NSTAGE - 1) % NSTAGE) * STAGE_ELEMS, M, (c + NSTAGE - 1) * CH,
                    rows, ld, col, tid, v16);
      cp_async_commit();
      const double *Sb = stages + (c % NSTAGE) * STAGE_ELEMS;
      double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const double a = Sb[(ks * 4 + (lane & 3)) * CHS + warp * 8 + (lane >> 2)];
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[j][0], acc[j][1], a, bz[j][ks]);
      }
      // rows of this chunk are read only from the stage: write straight back
      const int64_t row = c * CH + warp * 8 + (lane >> 2);
      if (row < rows) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int cc = col[j * 8 + 2 * (lane & 3) + h];
            if (cc >= 0) M[row + (int64_t)cc * ld] = acc[j][h];
          }
      }
    }
    cp_async_wait<0>();
  }
}

// Whole Jacobi iteration in one cooperative launch: sweeps x steps x pairs
// with a grid barrier between steps; the sweep's rotation count decides
// convergence on the device (no host round trip per sweep).  counters
// [max_sweeps] must be zero; status[0] receives the sweeps used (or -1).
// X is mX x n (ld ldx), P is n x n (ld ldp).
template <int NS>
__global__ void __launch_bounds__(JT, NS == 4 ? 2 : 3) k_jacobi_persistent(int64_t n, int64_t mX,
                                                          double *__restrict__ X, int64_t ldx,
                                                          double *__restrict__ P, int64_t ldp,
                                                          int nblk, double tol, double floor,
                                                          int max_sweeps, int csize,
                                                          unsigned long long *__restrict__ counters,
                                                          int *__restrict__ status,
                                                          int *__restrict__ last_mod,
                                                          int *__restrict__ last_ok) {
  __shared__ JacSmem sm;
  extern __shared__ __align__(16) double jac_stages[];
  cg::grid_group grid = cg::this_grid();
  const int npairs = nblk / 2;
  // csize CTAs (one cluster, or csize == 1) share a pair, each on a row slice
  const int cid = blockIdx.x / csize, crank = blockIdx.x % csize, ncl = gridDim.x / csize;
  for (int sw = 0; sw < max_sweeps; ++sw) {
    for (int step = 0; step < nblk - 1; ++step) {
      const JacTrack track{last_mod, last_ok, sw * (nblk - 1) + step};
      for (int pc = cid; pc < npairs; pc += ncl)
        jacobi_pair<NS>(n, mX, X, ldx, P, ldp, nblk, step, pc, tol, floor, counters + sw, sm, jac_stages,
                    crank, csize, &track);
      grid.sync();
    }
    const unsigned long long rot = *((volatile unsigned long long *)(counters + sw));
    if (rot == 0) {
      if (blockIdx.x == 0 && threadIdx.x == 0) status[0] = sw + 1;
      return;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) status[0] = -1;
}
// R (n x n, ld n, zero below the diagonal) from the factored A.
__global__ void k_upper(int64_t n, const double *__restrict__ A, int64_t lda, double *__restrict__ R) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / n, i = t - j * n;
    R[i + j * n] = i <= j ? A[i + j * lda] : 0.0;
  }
}

// V[piv[i], :] = W[i, :] (rows back to the original column order).
__global__ void k_unpivot_rows(int64_t n, int64_t r, const int *__restrict__ piv,
                               const double *__restrict__ W, int64_t ldw, double *__restrict__ V,
                               int64_t ldv) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * r;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / n, i = t - j * n;
    V[piv[i] + j * ldv] = W[i + j * ldw];
  }
}

// X = R^T from the factored A (upper triangle = R), n x n.
__global__ void k_rt(int64_t n, const double *__restrict__ A, int64_t lda, double *__restrict__ X) {
  int64_t total = n * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / n, i = t - j * n;  // X(i, j) = R(j, i) for j <= i
    X[i + j * n] = j <= i ? A[j + i * lda] : 0.0;
  }
}

__global__ void k_col_norms(int64_t n, int64_t ncol, const double *__restrict__ Y, int64_t ld,
                            double *__restrict__ out) {
  // one block per column, deterministic tree
  __shared__ double s[256];
  int64_t j = blockIdx.x;
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double v = Y[i + j * ld];
    a += v * v;
  }
  s[threadIdx.x] = a;
  __syncthreads();
  for (int off = blockDim.x / 2; off; off >>= 1) {
    if ((int)threadIdx.x < off) s[threadIdx.x] += s[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = sqrt(s[0]);
}

// out (rows x r): column j = src[:, sel[j]] * (scale ? 1/sig[j] : 1); rows beyond
// src_rows are zero.
__global__ void k_gather_cols(int64_t rows, int64_t src_rows, int64_t r, const double *__restrict__ src,
                              int64_t lds, const int64_t *__restrict__ sel,
                              const double *__restrict__ inv, double *__restrict__ out, int64_t ldo) {
  int64_t total = rows * r;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / rows, i = t - j * rows;
    double v = 0.0;
    if (i < src_rows) {
      v = src[i + sel[j] * lds];
      if (inv) v *= inv[j];
    }
    out[i + j * ldo] = v;
  }
}

// _fix_signs (linalg.py:56-63): first argmax |U[:, j]|; flip U[:, j] and
// V[:, j] if that entry is negative; then optionally V[:, j] *= s[j].
// k_sign_pick: one CTA per column decides the sign (fixed-order tree);
// k_sign_apply: grid (rank, chunks) rescales the rows (wide factors);
// k_sign_write: sign + layout in one pass (rank <= 32).
__global__ void k_sign_pick(int64_t mu, const double *__restrict__ U, int64_t ldu,
                            double *__restrict__ fac) {
  const int64_t j = blockIdx.x;
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  double best = -1.0;
  int64_t bi = 0;
  for (int64_t i = threadIdx.x; i < mu; i += blockDim.x) {
    double a = fabs(U[i + j * ldu]);
    if (a > best) {
      best = a;
      bi = i;
    }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int off = blockDim.x / 2; off; off >>= 1) {
    if ((int)threadIdx.x < off) {
      double o = sv[threadIdx.x + off];
      int64_t oi = si[threadIdx.x + off];
      if (o > sv[threadIdx.x] || (o == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = o;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) fac[j] = U[si[0] + j * ldu] < 0.0 ? -1.0 : 1.0;
}

// Sign rule + output layout in one pass: U_out = U fac, V_out = V fac
// (times sigma with scale_v), each written column- or row-major into the
// caller's buffer (replaces k_sign_apply + a transpose/copy per factor).
__global__ void k_sign_write(int64_t mu, int64_t mv, int64_t rank, const double *__restrict__ U,
                             const double *__restrict__ V, const double *__restrict__ fac,
                             const double *__restrict__ sig, int scale_v, double *__restrict__ Uo,
                             int64_t ldu, int u_row_major, double *__restrict__ Vo, int64_t ldv,
                             int v_row_major) {
  const int64_t nu = Uo ? mu * rank : 0, nv = Vo ? mv * rank : 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nu + nv;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < nu) {
      // row-major destination: consecutive threads write consecutive columns
      const int64_t i = u_row_major ? e / rank : e % mu, j = u_row_major ? e % rank : e / mu;
      const double v = fac[j] * U[i + j * mu];
      if (u_row_major) Uo[j + i * ldu] = v;
      else Uo[i + j * ldu] = v;
    } else {
      const int64_t f = e - nu;
      const int64_t i = v_row_major ? f / rank : f % mv, j = v_row_major ? f % rank : f / mv;
      const double v = fac[j] * (scale_v ? sig[j] : 1.0) * V[i + j * mv];
      if (v_row_major) Vo[j + i * ldv] = v;
      else Vo[i + j * ldv] = v;
    }
  }
}

__global__ void k_sign_apply(int64_t mu, int64_t mv, double *__restrict__ U, int64_t ldu,
                             double *__restrict__ V, int64_t ldv, const double *__restrict__ fac,
                             const double *__restrict__ sig, int scale_v) {
  const int64_t j = blockIdx.x;
  const double fu = fac[j];
  const double fv = fu * (scale_v ? sig[j] : 1.0);
  const int64_t nch = gridDim.y, c = blockIdx.y;
  const int64_t u0 = mu * c / nch, u1 = mu * (c + 1) / nch;
  const int64_t v0 = mv * c / nch, v1 = mv * (c + 1) / nch;
  if (fu != 1.0)
    for (int64_t i = u0 + threadIdx.x; i < u1; i += blockDim.x) U[i + j * ldu] = -U[i + j * ldu];
  if (fv != 1.0)
    for (int64_t i = v0 + threadIdx.x; i < v1; i += blockDim.x) V[i + j * ldv] *= fv;
}

}  // namespace

}  // namespace ftt

namespace ftt {
namespace {

// Deterministic test matrix for the low-rank range finder: splitmix64 of the
// element index, mapped to [-1, 1).
__global__ void k_omega(int64_t total, double *__restrict__ O) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)t + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    O[t] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
}

}  // namespace

void svd_state_release(ftt_ctx *ctx, SvdState *s) {
  if (!s) return;
  owned_free(ctx, s->Af);
  owned_free(ctx, s->tau);
  owned_free(ctx, s->Tb);
  if (!s->direct) owned_free(ctx, s->Y);
  owned_free(ctx, s->P);
  owned_free(ctx, s->B);
  owned_free(ctx, s->tau2);
  owned_free(ctx, s->Tb2);
  owned_free(ctx, s->piv);
  owned_free(ctx, s->Qk);
  owned_free(ctx, s->Bk);
  svd_state_release(ctx, s->inner);
  delete s;
}

void svd_state_free(ftt_ctx *ctx) {
  if (!ctx->svd) return;
  svd_state_release(ctx, ctx->svd);
  ctx->svd = nullptr;
}

namespace {

// Phase 1 (QR + Jacobi) on a given state; see the file header.
// extra_dev / extra_host: a device scalar of the caller brought back with
// the narrow path's single round trip (ignored on the wide path).
// allow_direct: the caller only uses singular triplets well above the noise
// floor (the low-rank path's inner factor), so the direct one-sided Jacobi on
// A_tall (U = Y / sigma) may be used for short narrow operands.
int svd_factor(ftt_ctx *ctx, SvdState *st, int64_t m, int64_t n, const double *A, int64_t lda,
               int32_t a_row_major, const double *extra_dev = nullptr,
               double *extra_host = nullptr, bool allow_direct = false, int extra_n = 1) {
  st->m = m;
  st->n = n;
  st->transposed = m < n;
  st->mA = std::max(m, n);
  st->nA = std::min(m, n);
  const int64_t mA = st->mA, nA = st->nA;
  if (nA == 0) return FTT_OK;
  static const bool no_small = getenv("FTT_NO_SMALL") != nullptr;
  // FTT_SVD_DIRECT=1: the direct path for every eligible operand (latency
  // probes of the inner-factor kernel through ftt_svd_f64)
  static const bool force_direct = getenv("FTT_SVD_DIRECT") != nullptr;
  if (!no_small && (allow_direct || force_direct) && direct_small_ok(mA, nA)) {
    // short narrow operand (e.g. the k x n_A factor B of the low-rank path):
    // the narrow path's factorisation in one CTA (Householder QR in shared
    // memory, Jacobi on R^T, U = Q P); phase 2 takes the `small` branch
    st->small = true;
    const bool need_t = a_row_major ? !st->transposed : st->transposed;
    FTT_CHECK(owned_alloc(ctx, (void **)&st->Af, 8 * (size_t)mA * nA));
    FTT_CHECK(owned_alloc(ctx, (void **)&st->Y, 8 * (size_t)nA * nA));
    std::vector<double> raw(nA);
    const int pb = prof_begin(ctx);
    FTT_CHECK(direct_small_svd(ctx, mA, nA, A, lda, need_t ? 1 : 0, st->Af, st->Y, raw.data(),
                               &st->sweeps, extra_dev, extra_host, extra_n));
    // QR (2 m n^2) + Q P (2 m n^2) + sweeps x n^2/2 pairs x 6 n
    prof_end(ctx, pb, PT_JACOBI, 8.0 * ((double)mA * nA * 2 + (double)nA * nA),
             4.0 * (double)mA * nA * nA + 3.0 * std::max(st->sweeps, 1) * (double)nA * nA * nA);
    st->perm.resize(nA);
    std::iota(st->perm.begin(), st->perm.end(), 0);
    std::stable_sort(st->perm.begin(), st->perm.end(),
                     [&](int64_t a, int64_t b) { return raw[a] > raw[b]; });
    st->sigma.resize(nA);
    for (int64_t i = 0; i < nA; ++i) st->sigma[i] = raw[st->perm[i]];
    return FTT_OK;
  }
  if (!no_small && tsqr_ok(mA, nA)) {
    // narrow operand: CTA-local QR (+ TSQR tree) and CTA-local Jacobi, one
    // host round trip for the whole factorisation
    st->small = true;
    const bool need_t = a_row_major ? !st->transposed : st->transposed;
    FTT_CHECK(owned_alloc(ctx, (void **)&st->Af, 8 * (size_t)mA * nA));
    FTT_CHECK(owned_alloc(ctx, (void **)&st->Y, 8 * (size_t)nA * nA));
    std::vector<double> raw(nA);
    const int pb = prof_begin(ctx);
    FTT_CHECK(tsqr_svd(ctx, mA, nA, A, lda, need_t ? 1 : 0, st->Af, mA, st->Y, raw.data(),
                       &st->sweeps, extra_dev, extra_host, extra_n));
    // QR (4 m n^2 / 3) + Q formation + Q P, plus sweeps x n^2/2 pairs x 10 n
    prof_end(ctx, pb, PT_JACOBI, 8.0 * ((double)mA * nA * 3 + (double)nA * nA * 2),
             (double)mA * nA * nA * (8.0 / 3.0 + 2.0) + 5.0 * std::max(st->sweeps, 1) *
                                                           (double)nA * nA * nA);
    static const bool debug = getenv("FTT_DEBUG") != nullptr;
    if (debug)
      fprintf(stderr, "[ftt] svd m=%lld n=%lld (mA=%lld nA=%lld small) sweeps %d\n", (long long)m,
              (long long)n, (long long)mA, (long long)nA, st->sweeps);
    st->perm.resize(nA);
    std::iota(st->perm.begin(), st->perm.end(), 0);
    std::stable_sort(st->perm.begin(), st->perm.end(),
                     [&](int64_t a, int64_t b) { return raw[a] > raw[b]; });
    st->sigma.resize(nA);
    for (int64_t i = 0; i < nA; ++i) st->sigma[i] = raw[st->perm[i]];
    return FTT_OK;
  }
  {
    FTT_CHECK(arena_reserve(ctx, 1024));
    bool ok = true;
    if (a_row_major) FTT_CHECK(check_finite(ctx, n, m, A, lda, &ok));
    else FTT_CHECK(check_finite(ctx, m, n, A, lda, &ok));
    if (!ok) {
      set_error("matrix entries must be finite");
      return FTT_ERR_NONFINITE;
    }
  }
  FTT_CHECK(owned_alloc(ctx, (void **)&st->Af, 8 * (size_t)mA * nA));
  FTT_CHECK(owned_alloc(ctx, (void **)&st->tau, 8 * (size_t)nA));
  FTT_CHECK(owned_alloc(ctx, (void **)&st->Tb, 8 * qr_tblk_elems(mA, nA)));
  // Direct mode (opt-in, FTT_DIRECT=1): one-sided Jacobi on A_tall itself
  // for nearly square operands.  Measured slower on the low-rank operands of
  // the BASELINE configs (the QR concentrates the rank into a few rows of R,
  // so most columns of R^T start near the noise floor), hence off by default.
  {
    static const char *dm = getenv("FTT_DIRECT");
    st->direct = dm && dm[0] == '1' && nA > 1 && mA <= 3 * nA;
  }
  {
    static const char *pc = getenv("FTT_PRECOND");
    st->precond = !st->direct && nA > 1 && pc && pc[0] == '1';  // off by default
    // pivoted QR of R before the Jacobi (FTT_QRCP=0 off, =1 for every
    // size): on by default for 96..1024 columns, where R stays L2-resident
    // and the BLAS-2 pivoted factorization costs a few ms (config 4's
    // 2064 x 766 operand: Jacobi 88 -> 33 ms incl. the QRCP).  Wider
    // operands are left unpivoted: on config 3's 25168 x 4916 operand the
    // QRCP streams R from HBM every step (~0.6 s) and its more accurate small
    // singular values moved a tail decision away from LAPACK gesdd's
    // (rank 1975 vs the reference's 1971).
    static const char *qp = getenv("FTT_QRCP");
    const bool qp_all = qp && qp[0] == '1', qp_off = qp && qp[0] == '0';
    st->pivoted = !st->direct && !st->precond && !qp_off && qrcp_ok(nA) && nA >= 96 &&
                  (qp_all || nA <= 1024);
  }
  if (!st->direct) FTT_CHECK(owned_alloc(ctx, (void **)&st->Y, 8 * (size_t)nA * nA));
  FTT_CHECK(owned_alloc(ctx, (void **)&st->P, 8 * (size_t)nA * nA));
  if (st->precond || st->pivoted) {
    FTT_CHECK(owned_alloc(ctx, (void **)&st->B, 8 * (size_t)nA * nA));
    FTT_CHECK(owned_alloc(ctx, (void **)&st->tau2, 8 * (size_t)nA));
    FTT_CHECK(owned_alloc(ctx, (void **)&st->Tb2, 8 * qr_tblk_elems(nA, nA)));
  }
  if (st->pivoted) FTT_CHECK(owned_alloc(ctx, (void **)&st->piv, 4 * (size_t)nA));
  // tall orientation A_tall (mA x nA, column-major): M itself when m >= n,
  // else M^T.  A row-major M is the column-major M^T.
  const bool need_t = a_row_major ? !st->transposed : st->transposed;
  if (!need_t) {
    FTT_CHECK(copy_matrix(ctx, mA, nA, A, lda, st->Af, mA));
  } else {
    FTT_CHECK(transpose(ctx, nA, mA, A, lda, st->Af, mA));
  }
  size_t wse = qr_workspace_elems(mA, nA);
  const int64_t nblk_max = ceil_div(nA, JB) + 1;
  FTT_CHECK(arena_reserve(ctx, align_up(8 * wse) + align_up(8 * (size_t)nA) +
                                   align_up(8 * (kSumSqBlocks + 1)) +
                                   align_up(4 * nblk_max * (nblk_max + 1)) + 4096));
  double *ws = take<double>(ctx, wse);
  double *norms = take<double>(ctx, nA);
  double *partial = take<double>(ctx, kSumSqBlocks + 1);
  unsigned long long *rot = take<unsigned long long>(ctx, 64);
  int *track_buf = take<int>(ctx, nblk_max * (nblk_max + 1));
  static const bool debug = getenv("FTT_DEBUG") != nullptr;
  cudaEvent_t dbg_ev[3];
  if (debug) {
    for (auto &e : dbg_ev) cudaEventCreate(&e);
    cudaEventRecord(dbg_ev[0], ctx->stream);
  }
  if (!st->direct) FTT_CHECK(qr_factor(ctx, mA, nA, st->Af, mA, st->tau, st->Tb, ws, wse));
  if (debug) cudaEventRecord(dbg_ev[1], ctx->stream);
  if (st->direct) {
    st->Y = st->Af;  // Jacobi on A_tall (mA x nA) in place
  } else if (st->precond) {
    // R^T = Q2 R2, Jacobi on X = R2^T; A = (Q Yhat) Sigma (Q2 P)^T
    k_rt<<<grid_for(nA * nA, 256, 4), 256, 0, ctx->stream>>>(nA, st->Af, mA, st->B);
    FTT_LAUNCHED(ctx);
    FTT_CHECK(qr_factor(ctx, nA, nA, st->B, nA, st->tau2, st->Tb2, ws, wse));
    k_rt<<<grid_for(nA * nA, 256, 4), 256, 0, ctx->stream>>>(nA, st->B, nA, st->Y);
    FTT_LAUNCHED(ctx);
  } else if (st->pivoted) {
    // R (upper triangle of the factored A) -> R Pi = Q2 R2 -> X = R2^T
    k_upper<<<grid_for(nA * nA, 256, 4), 256, 0, ctx->stream>>>(nA, st->Af, mA, st->Y);
    FTT_LAUNCHED(ctx);
    FTT_CHECK(qrcp_factor(ctx, nA, st->Y, st->B, st->tau2, st->piv));
    FTT_CHECK(qr_build_tblk(ctx, nA, nA, st->B, nA, st->tau2, st->Tb2, ws, wse));
    k_rt<<<grid_for(nA * nA, 256, 4), 256, 0, ctx->stream>>>(nA, st->B, nA, st->Y);
    FTT_LAUNCHED(ctx);
  } else {
    k_rt<<<grid_for(nA * nA, 256, 4), 256, 0, ctx->stream>>>(nA, st->Af, mA, st->Y);
    FTT_LAUNCHED(ctx);
  }
  FTT_CHECK(launch_identity(ctx, nA, nA, st->P, nA));
  const int64_t mX = st->direct ? mA : nA;
  if (nA > 1) {
    int nblk = (int)ceil_div(nA, JB);
    if (nblk & 1) ++nblk;
    // relative orthogonality target sqrt(n) eps (LAPACK dgesvj's);
    // (scaling it up to 16x was measured to leave the sweep counts unchanged)
    const double tol = 2.220446049250313e-16 * sqrt((double)nA);
    // noise floor: columns with |x|^2 <= (0.1 eps)^2 * rows * ||X||_F^2 are
    // below the backward error of the QR and are not orthogonalised further
    double fro2 = 0.0;
    FTT_CHECK(sum_squares(ctx, mX * nA, st->Y, partial, &fro2));
    const double floor = 0.01 * 2.220446049250313e-16 * 2.220446049250313e-16 * (double)mX * fro2;
    const int max_sweeps = 60;
    FTT_CUDA(cudaMemsetAsync(rot, 0, sizeof(unsigned long long) * 64, ctx->stream));
    static int coresident = 0, coresident3 = 0;
    if (!coresident) {
      int per_sm = 0, per_sm3 = 0;
      FTT_CUDA(cudaFuncSetAttribute(k_jacobi_persistent<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)jac_dyn_bytes(4)));
      FTT_CUDA(cudaFuncSetAttribute(k_jacobi_persistent<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)jac_dyn_bytes(3)));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi_persistent<4>, JT, jac_dyn_bytes(4));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm3, k_jacobi_persistent<3>, JT, jac_dyn_bytes(3));
      coresident = std::max(1, per_sm) * ctx->num_sms;
      coresident3 = std::max(1, per_sm3) * ctx->num_sms;
    }
    // Pairs are split over a cluster of csize CTAs (row slices, DSMEM Gram
    // sum) when there are fewer pairs than co-resident CTAs: each slice
    // keeps >= 3 chunks of 64 rows (config 4: 4-CTA clusters 165 -> 131 ms).
    // Between coresident/2 and coresident3/2 pairs (e.g. config 3's 154) the
    // 3-stage / 3-CTAs-per-SM variant runs 2-CTA clusters instead of leaving
    // a few SMs with two whole pairs (~10 % per sweep).  FTT_JCLUSTER=c
    // forces c (1 = off).
    const int npairs = nblk / 2;
    static const int cs_env = getenv("FTT_JCLUSTER") ? atoi(getenv("FTT_JCLUSTER")) : 0;
    int csize = cs_env > 0 ? std::min(8, cs_env)
                           : (int)std::max<int64_t>(1, std::min<int64_t>({8, coresident / std::max(1, npairs),
                                                                          ceil_div(mX, CH) / 3}));
    int ns = 4;
    if (cs_env <= 0 && csize == 1 && 2 * npairs > coresident && 2 * npairs <= coresident3 &&
        ceil_div(mX, CH) >= 6) {
      ns = 3;
      csize = 2;
    }
    const void *kfn =
        ns == 4 ? (const void *)k_jacobi_persistent<4> : (const void *)k_jacobi_persistent<3>;
    int G = std::min(npairs, ns == 4 ? coresident : coresident3);
    cudaLaunchAttribute lattr[2];
    lattr[0].id = cudaLaunchAttributeCooperative;
    lattr[0].val.cooperative = 1;
    lattr[1].id = cudaLaunchAttributeClusterDimension;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(JT);
    cfg.dynamicSmemBytes = jac_dyn_bytes(ns);
    cfg.stream = ctx->stream;
    cfg.attrs = lattr;
    cfg.numAttrs = 1;
    if (csize > 1) {
      lattr[1].val.clusterDim.x = csize;
      lattr[1].val.clusterDim.y = 1;
      lattr[1].val.clusterDim.z = 1;
      cfg.numAttrs = 2;
      cfg.gridDim = dim3(npairs * csize);
      int maxc = 0;
      if (cudaOccupancyMaxActiveClusters(&maxc, kfn, &cfg) != cudaSuccess ||
          maxc < 1) {
        cudaGetLastError();
        csize = 1;
        cfg.numAttrs = 1;
      } else {
        G = std::min(npairs, maxc) * csize;
      }
    }
    cfg.gridDim = dim3(G);
    g_last_csize = csize;
    int64_t nA_ = nA, mX_ = mX;
    double *Y = st->Y, *Pm = st->P;
    int nblk_ = nblk;
    double tol_ = tol, floor_ = floor;
    int maxsw = max_sweeps;
    unsigned long long *cnt = rot;
    int *status = reinterpret_cast<int *>(rot + max_sweeps);
    // last_mod[nblk] = -1 (0xff bytes), last_ok[nblk*nblk] = -1: nothing verified yet
    int *last_mod = track_buf;
    int *last_ok = track_buf + nblk;
    FTT_CUDA(cudaMemsetAsync(track_buf, 0xff, sizeof(int) * (size_t)nblk * (nblk + 1), ctx->stream));
    void *args[] = {&nA_, &mX_, &Y, &mX_, &Pm, &nA_, &nblk_, &tol_, &floor_, &maxsw, &csize, &cnt,
                    &status, &last_mod, &last_ok};
    const int pb = prof_begin(ctx);
    cudaError_t le = cudaLaunchKernelExC(&cfg, kfn, args);
    if (le != cudaSuccess && csize > 1) {
      // a cooperative launch of clusters refused (e.g. under a replaying
      // profiler): the same iteration with one CTA per pair
      cudaGetLastError();
      csize = 1;
      g_last_csize = 1;
      kfn = (const void *)k_jacobi_persistent<4>;
      cfg.numAttrs = 1;
      cfg.dynamicSmemBytes = jac_dyn_bytes(4);
      cfg.gridDim = dim3(std::min(npairs, coresident));
      le = cudaLaunchKernelExC(&cfg, kfn, args);
    }
    FTT_CUDA(le);
    FTT_LAUNCHED(ctx);
    int sw_used = 0;
    FTT_CHECK(copy_to_host(ctx, &sw_used, status, sizeof(int)));
    // per sweep and step: every block pair forms its 32x32 Gram from X
    // (2*32^2*mX flops) and applies the rotation to X and P (2*32^2*(mX+n))
    const double sweeps_d = sw_used > 0 ? sw_used : max_sweeps;
    prof_end(ctx, pb, PT_JACOBI, sweeps_d * (nblk - 1) * 8.0 * (3.0 * mX + 2.0 * nA) * nA,
             sweeps_d * (nblk - 1) * (nblk / 2) * 2.0 * JP * JP * (2.0 * mX + (double)nA));
    st->sweeps = sw_used;
    if (sw_used < 0) {
      set_error("Jacobi SVD did not converge in %d sweeps", max_sweeps);
      return FTT_ERR_NOCONV;
    }
  }
  if (debug) {
    cudaEventRecord(dbg_ev[2], ctx->stream);
    cudaEventSynchronize(dbg_ev[2]);
    float qr_ms = 0, jac_ms = 0;
    cudaEventElapsedTime(&qr_ms, dbg_ev[0], dbg_ev[1]);
    cudaEventElapsedTime(&jac_ms, dbg_ev[1], dbg_ev[2]);
    fprintf(stderr, "[ftt] svd m=%lld n=%lld (mA=%lld nA=%lld%s) qr %.3f ms jacobi %.3f ms sweeps %d",
            (long long)m, (long long)n, (long long)mA, (long long)nA, st->direct ? " direct" : "",
            qr_ms, jac_ms, st->sweeps);
    fprintf(stderr, " cluster %d", g_last_csize);
    if (st->sweeps > 0) {
      std::vector<unsigned long long> cnt(st->sweeps);
      cudaMemcpy(cnt.data(), rot, 8 * st->sweeps, cudaMemcpyDeviceToHost);
      fprintf(stderr, " rotated pairs/sweep:");
      for (auto c : cnt) fprintf(stderr, " %llu", c);
    }
    fprintf(stderr, "\n");
    for (auto &e : dbg_ev) cudaEventDestroy(e);
  }
  k_col_norms<<<(unsigned)nA, 256, 0, ctx->stream>>>(mX, nA, st->Y, mX, norms);
  FTT_LAUNCHED(ctx);
  std::vector<double> raw(nA);
  FTT_CHECK(copy_to_host(ctx, raw.data(), norms, 8 * nA));
  st->perm.resize(nA);
  std::iota(st->perm.begin(), st->perm.end(), 0);
  std::stable_sort(st->perm.begin(), st->perm.end(),
                   [&](int64_t a, int64_t b) { return raw[a] > raw[b]; });
  st->sigma.resize(nA);
  for (int64_t i = 0; i < nA; ++i) st->sigma[i] = raw[st->perm[i]];
  return FTT_OK;
}

// The leading `rank` triplets of a full (non-low-rank) state in its tall
// orientation: UA (mA x rank), VA (nA x rank), column-major, unscaled and
// without the sign rule.
// sig_host (optional): rank values staged with the selection in the same
// host->device copy; *sig_dev receives their device address, followed by
// rank doubles of device scratch.
int svd_raw_vectors(ftt_ctx *ctx, SvdState *st, int64_t rank, double *UA, double *VA,
                    const double *sig_host = nullptr, double **sig_dev = nullptr) {
  const int64_t mA = st->mA, nA = st->nA;
  size_t wse = qr_apply_workspace_elems(mA, nA, rank);
  FTT_CHECK(arena_reserve(ctx, align_up(8 * wse) + align_up(8 * 4 * rank) + 4096));
  double *ws = take<double>(ctx, wse);
  // one staged copy: [sel (int64) | 1/sigma | sig_host], then scratch
  double *packed = take<double>(ctx, 4 * rank);
  int64_t *sel = reinterpret_cast<int64_t *>(packed);
  double *inv = packed + rank;
  std::vector<double> h(3 * rank);
  memcpy(h.data(), st->perm.data(), 8 * rank);
  for (int64_t j = 0; j < rank; ++j) h[rank + j] = st->sigma[j] != 0.0 ? 1.0 / st->sigma[j] : 0.0;
  const int64_t nst = sig_host ? 3 * rank : 2 * rank;
  if (sig_host) {
    memcpy(h.data() + 2 * rank, sig_host, 8 * rank);
    *sig_dev = packed + 2 * rank;
  }
  FTT_CHECK(stage_to_device(ctx, packed, h.data(), 8 * nst));
  if (st->small) {
    // U_A = (Q P)[:, sel],  V_A = Y[:, sel] / sigma
    k_gather_cols<<<grid_for(mA * rank, 256, 4), 256, 0, ctx->stream>>>(mA, mA, rank, st->Af, mA,
                                                                        sel, nullptr, UA, mA);
    FTT_LAUNCHED(ctx);
    k_gather_cols<<<grid_for(nA * rank, 256, 4), 256, 0, ctx->stream>>>(nA, nA, rank, st->Y, nA,
                                                                        sel, inv, VA, nA);
    FTT_LAUNCHED(ctx);
    return FTT_OK;
  }
  if (st->direct) {
    // U_A = Y[:, sel] / sigma (Y = A P, mA x nA),  V_A = P[:, sel]
    k_gather_cols<<<grid_for(mA * rank, 256, 4), 256, 0, ctx->stream>>>(mA, mA, rank, st->Y, mA,
                                                                        sel, inv, UA, mA);
    FTT_LAUNCHED(ctx);
    k_gather_cols<<<grid_for(nA * rank, 256, 4), 256, 0, ctx->stream>>>(nA, nA, rank, st->P, nA,
                                                                        sel, nullptr, VA, nA);
    FTT_LAUNCHED(ctx);
  } else if (st->precond) {
    // U_A = Q [Y[:, sel] / sigma; 0],  V_A = Q2 P[:, sel]
    k_gather_cols<<<grid_for(mA * rank, 256, 4), 256, 0, ctx->stream>>>(mA, nA, rank, st->Y, nA,
                                                                        sel, inv, UA, mA);
    FTT_LAUNCHED(ctx);
    k_gather_cols<<<grid_for(nA * rank, 256, 4), 256, 0, ctx->stream>>>(nA, nA, rank, st->P, nA,
                                                                        sel, nullptr, VA, nA);
    FTT_LAUNCHED(ctx);
    FTT_CHECK(qr_apply_q(ctx, nA, nA, st->B, nA, st->Tb2, rank, VA, nA, ws, wse));
  } else if (st->pivoted) {
    // A Pi = (Q Q2) R2, R2 = P Sigma Yhat^T:  V_A = Pi Yhat[:, sel],
    // U_A = Q [Q2 P[:, sel]; 0]
    double *W = nullptr;
    FTT_CHECK(owned_alloc(ctx, (void **)&W, 8 * (size_t)nA * rank));
    k_gather_cols<<<grid_for(nA * rank, 256, 4), 256, 0, ctx->stream>>>(nA, nA, rank, st->Y, nA,
                                                                        sel, inv, W, nA);
    FTT_LAUNCHED(ctx);
    k_unpivot_rows<<<grid_for(nA * rank, 256, 4), 256, 0, ctx->stream>>>(nA, rank, st->piv, W, nA,
                                                                         VA, nA);
    FTT_LAUNCHED(ctx);
    owned_free(ctx, W);
    k_gather_cols<<<grid_for(mA * rank, 256, 4), 256, 0, ctx->stream>>>(mA, nA, rank, st->P, nA,
                                                                        sel, nullptr, UA, mA);
    FTT_LAUNCHED(ctx);
    FTT_CHECK(qr_apply_q(ctx, nA, nA, st->B, nA, st->Tb2, rank, UA, mA, ws, wse));
  } else {
    // V_A = Y[:, sel] / sigma ;  U_A = Q [P[:, sel]; 0]
    k_gather_cols<<<grid_for(nA * rank, 256, 4), 256, 0, ctx->stream>>>(nA, nA, rank, st->Y, nA,
                                                                        sel, inv, VA, nA);
    FTT_LAUNCHED(ctx);
    k_gather_cols<<<grid_for(mA * rank, 256, 4), 256, 0, ctx->stream>>>(mA, nA, rank, st->P, nA,
                                                                        sel, nullptr, UA, mA);
    FTT_LAUNCHED(ctx);
  }
  if (!st->direct) FTT_CHECK(qr_apply_q(ctx, mA, nA, st->Af, mA, st->Tb, rank, UA, mA, ws, wse));
  return FTT_OK;
}

}  // namespace
}  // namespace ftt

using namespace ftt;

extern "C" int ftt_svd_f64(ftt_ctx *ctx, int64_t m, int64_t n, const double *A, int64_t lda,
                           int32_t a_row_major, double *s_host) {
  if (!ctx || m < 0 || n < 0) return FTT_ERR_INVALID;
  ctx->fro2_hint = 0.0;
  ctx->rank_hint = 0;
  svd_state_free(ctx);
  SvdState *st = new SvdState();
  ctx->svd = st;
  FTT_CHECK(svd_factor(ctx, st, m, n, A, lda, a_row_major));
  if (s_host && st->nA) memcpy(s_host, st->sigma.data(), 8 * st->nA);
  return FTT_OK;
}

// The certified low-rank path on a dense operand (A, lda, a_row_major) or on
// the entries of a sparse one (sp != nullptr, ftt_sparse.cu).
static int lowrank_run(ftt_ctx *ctx, int64_t m, int64_t n, const double *A, int64_t lda,
                       int32_t a_row_major, SparseOperand *sp, int64_t k, double delta2,
                       double *s_host, double *rest2_host, int32_t *accepted,
                       ScatterOperand *sc = nullptr) {
  if (!ctx || m < 0 || n < 0 || !accepted || !rest2_host) return FTT_ERR_INVALID;
  // ||A||_F^2 when the caller knows it (consumed here)
  const double fro2_known = ctx->fro2_hint;
  ctx->fro2_hint = 0.0;
  const int64_t rank_hint = ctx->rank_hint;
  ctx->rank_hint = 0;
  const bool have_fro2 = fro2_known > 0.0 && std::isfinite(fro2_known);
  svd_state_free(ctx);
  SvdState *st = new SvdState();
  ctx->svd = st;
  st->lowrank = true;
  st->m = m;
  st->n = n;
  st->transposed = m < n;
  st->mA = std::max(m, n);
  st->nA = std::min(m, n);
  const int64_t mA = st->mA, nA = st->nA;
  *accepted = 0;
  *rest2_host = -1.0;
  if (nA == 0 || k <= 0 || k >= nA) return FTT_OK;
  if ((sp || sc) && k > 64) return FTT_OK;  // sparse products handle sketches <= 64 wide
  // The tall view A_tall (mA x nA) is read straight from the caller's buffer:
  // `buf` col-major with leading dimension `ld`, stored transposed when
  // `need_t`.  A strided (non-packed) input is packed once first.
  const bool need_t = a_row_major ? !st->transposed : st->transposed;
  const double *buf = A;
  int64_t ld = lda;
  double fro2 = 0.0, rest2 = 0.0;
  // ||A||_F^2 stays on the device until the sketch rank comes back (one host
  // round trip for both); a non-finite entry is diagnosed there
  double *fro2_dev = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&fro2_dev, 8 * (size_t)(kSumSqBlocks + 6)));
  // after sum_squares' partials: rest2 | sketch rank word | ||A||_F^2 (read
  // back together)
  double *rest2_dev = fro2_dev + kSumSqBlocks + 2;
  double *fro2_out = rest2_dev + 2;
  if (sc) {
    if (!have_fro2) {
      if (sc->ldv != sc->K) {
        set_error("scattered operand: strided carry without a known norm");
        return FTT_ERR_INVALID;
      }
      FTT_CHECK(sum_squares_dev(ctx, sc->K * sc->r, sc->V, fro2_dev + 1, fro2_out));
    }
  } else if (sp) {
    if (!have_fro2)
      FTT_CHECK(sum_squares_dev(ctx, sp->nnz, sp->by_fiber ? sp->f_vals : sp->v_r, fro2_dev + 1,
                                fro2_out));
  } else {
    const int64_t inner = need_t ? nA : mA;
    if (lda != inner) {
      FTT_CHECK(owned_alloc(ctx, (void **)&st->Af, 8 * (size_t)mA * nA));
      FTT_CHECK(copy_matrix(ctx, inner, mA * nA / inner, A, lda, st->Af, inner));
      buf = st->Af;
      ld = inner;
    }
    if (!have_fro2) FTT_CHECK(sum_squares_dev(ctx, mA * nA, buf, fro2_dev + 1, fro2_out));
  }
  auto finite_or_decline = [&]() -> int {
    // non-finite energy: either a non-finite entry (error) or an overflow
    if (sp || sc) return FTT_OK;  // entries are validated finite: overflow, full SVD decides
    bool ok = true;
    FTT_CHECK(check_finite(ctx, need_t ? nA : mA, need_t ? mA : nA, buf, ld, &ok));
    if (!ok) {
      set_error("matrix entries must be finite");
      return FTT_ERR_NONFINITE;
    }
    return FTT_OK;  // not accepted: the caller takes the full SVD
  };
  double *Om = nullptr, *Yk = nullptr, *sk = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&Yk, 8 * (size_t)mA * k));
  FTT_CHECK(owned_alloc(ctx, (void **)&st->Qk, 8 * (size_t)mA * k));
  FTT_CHECK(owned_alloc(ctx, (void **)&st->Bk, 8 * (size_t)k * nA));
  const size_t ske = (sp || sc) ? 1 : std::max({gemm_splitk_elems(mA, k, nA), gemm_splitk_elems(k, nA, mA),
                                        gemm_splitk_elems(mA, nA, k), (size_t)1});
  FTT_CHECK(owned_alloc(ctx, (void **)&sk, 8 * ske));
  // range finder: Y = A Omega, Q = qr(Y), B = Q^T A, residual A - Q B (in place)
  if (sc) {
    FTT_CHECK(scatter_sketch(ctx, *sc, k, Yk));
  } else if (sp) {
    FTT_CHECK(sparse_sketch(ctx, *sp, k, Yk));
  } else {
    FTT_CHECK(owned_alloc(ctx, (void **)&Om, 8 * (size_t)nA * k));
    k_omega<<<grid_for(nA * k, 256, 4), 256, 0, ctx->stream>>>(nA * k, Om);
    FTT_LAUNCHED(ctx);
    FTT_CHECK(gemm(ctx, need_t, 0, mA, k, nA, 1.0, buf, ld, Om, nA, 0.0, Yk, mA, sk, ske));
  }
  static const char *qr_mode = getenv("FTT_SKETCH_QR");  // test override: householder
  static const bool no_speculate = getenv("FTT_NO_SPECULATE") != nullptr;
  static const bool no_rank_spec = getenv("FTT_NO_RANK_SPEC") != nullptr;
  const bool small_qr = k <= 64 && !(qr_mode && !strcmp(qr_mode, "householder"));
  int64_t *sel = nullptr;
  auto bail = [&]() {
    owned_free(ctx, sel);
    owned_free(ctx, Om);
    owned_free(ctx, Yk);
    owned_free(ctx, sk);
    owned_free(ctx, fro2_dev);
  };
  // Range basis from the kr spanning sketch columns, B = Q^T A, the
  // certificate residual and (narrow B) its factorisation, speculatively,
  // before the certificate is read: residual energy, singular values and --
  // when the sketch rank was assumed (rank_spec) -- the rank word and
  // ||A||_F^2 all come back in the inner factorisation's one round trip.
  bool rank_spec = false;
  double extras[3] = {0.0, 0.0, 0.0};  // rest2 | rank word | ||A||_F^2
  auto project = [&](int64_t kr) -> int {
    if (small_qr) {
      double *Ys = nullptr;
      FTT_CHECK(owned_alloc(ctx, (void **)&Ys, 8 * (size_t)mA * kr));
      k_gather_cols<<<grid_for(mA * kr, 256, 4), 256, 0, ctx->stream>>>(mA, mA, kr, Yk, mA, sel,
                                                                        nullptr, Ys, mA);
      FTT_LAUNCHED(ctx);
      FTT_CHECK(tsqr_q(ctx, mA, kr, Ys, mA, 0, st->Qk, mA, nullptr, 0, false));
      owned_free(ctx, Ys);
    }
    if (sc) FTT_CHECK(scatter_qt_a(ctx, *sc, kr, st->Qk, st->Bk));
    else if (sp) FTT_CHECK(sparse_qt_a(ctx, *sp, kr, st->Qk, st->Bk));
    else FTT_CHECK(gemm(ctx, 1, need_t, kr, nA, mA, 1.0, st->Qk, mA, buf, ld, 0.0, st->Bk, kr, sk,
                        ske));
    const bool speculate = tsqr_ok(std::max(kr, nA), std::min(kr, nA)) && !no_speculate;
    if (speculate) {
      if (sc) FTT_CHECK(scatter_resid(ctx, *sc, kr, st->Qk, st->Bk, rest2_dev));
      else if (sp) FTT_CHECK(sparse_resid(ctx, *sp, kr, st->Qk, st->Bk, rest2_dev));
      else FTT_CHECK(gemm_resid_sumsq(ctx, 0, 0, mA, nA, kr, st->Qk, mA, st->Bk, kr, buf, ld,
                                      need_t, nullptr, rest2_dev));
      st->inner = new SvdState();
      if (svd_factor(ctx, st->inner, kr, nA, st->Bk, kr, 0, rest2_dev, extras, true,
                     rank_spec ? 3 : 1) != FTT_OK) {
        // speculative factorisation failed: decide on the certificate alone
        // (an accepted certificate re-runs the factorisation below and reports)
        svd_state_release(ctx, st->inner);
        st->inner = nullptr;
        FTT_CHECK(copy_to_host(ctx, extras, rest2_dev, (rank_spec ? 3 : 1) * sizeof(double)));
      }
      rest2 = extras[0];
    } else if (sp || sc) {
      if (sc) FTT_CHECK(scatter_resid(ctx, *sc, kr, st->Qk, st->Bk, rest2_dev));
      else FTT_CHECK(sparse_resid(ctx, *sp, kr, st->Qk, st->Bk, rest2_dev));
      FTT_CHECK(copy_to_host(ctx, extras, rest2_dev, (rank_spec ? 3 : 1) * sizeof(double)));
      rest2 = extras[0];
    } else {
      FTT_CHECK(gemm_resid_sumsq(ctx, 0, 0, mA, nA, kr, st->Qk, mA, st->Bk, kr, buf, ld, need_t,
                                 &rest2));
      if (rank_spec) FTT_CHECK(copy_to_host(ctx, extras, rest2_dev, 3 * sizeof(double)));
    }
    return FTT_OK;
  };
  if (small_qr) {
    // numerical rank of the sketch (pivoted Cholesky of its Gram, directions
    // below ~3e-6 of the largest dropped -- the residual certificate decides
    // whether the basis suffices), then Householder TSQR of only the r
    // spanning columns (ftt_cholqr.cu, ftt_small.cu).  With the caller's
    // rank hint the rank word is not waited for: the step runs at the hinted
    // rank and is redone at the true one if they differ.
    int64_t kr = 0;
    FTT_CHECK(owned_alloc(ctx, (void **)&sel, 8 * (size_t)k));
    rank_spec = ctx->spec_ok && !no_rank_spec && rank_hint > 0 && rank_hint <= k &&
                rank_hint < nA;
    if (rank_spec) {
      FTT_CUDA(cudaMemsetAsync(rest2_dev + 1, 0, 8, ctx->stream));
      FTT_CHECK(sketch_rank_async(ctx, mA, k, Yk, 1e-11, sel,
                                  reinterpret_cast<int *>(rest2_dev + 1)));
      kr = rank_hint;
      FTT_CHECK(project(kr));
      int kr_true = 0;
      memcpy(&kr_true, &extras[1], sizeof(int));
      fro2 = have_fro2 ? fro2_known : extras[2];
      if (kr_true != kr || !std::isfinite(fro2)) {
        // wrong guess: no further guesses in this sweep; redo at the true rank
        ctx->spec_ok = false;
        rank_spec = false;
        if (st->inner) {
          svd_state_release(ctx, st->inner);
          st->inner = nullptr;
        }
        kr = kr_true;
        if (kr == 0 || !std::isfinite(fro2)) {
          bail();
          return std::isfinite(fro2) ? FTT_OK : finite_or_decline();  // full SVD instead
        }
        FTT_CHECK(project(kr));
      }
    } else {
      FTT_CHECK(sketch_rank(ctx, mA, k, Yk, 1e-11, sel, &kr, have_fro2 ? nullptr : fro2_out, &fro2));
      if (have_fro2) fro2 = fro2_known;
      if (kr == 0 || !std::isfinite(fro2)) {
        bail();
        return std::isfinite(fro2) ? FTT_OK : finite_or_decline();  // full SVD instead
      }
      FTT_CHECK(project(kr));
    }
    owned_free(ctx, sel);
    sel = nullptr;
    k = kr;
  } else {
    if (have_fro2) fro2 = fro2_known;
    else FTT_CHECK(copy_to_host(ctx, &fro2, fro2_out, sizeof(double)));
    if (!std::isfinite(fro2)) {
      bail();
      return finite_or_decline();
    }
    size_t wse = qr_workspace_elems(mA, k);
    FTT_CHECK(arena_reserve(ctx, align_up(8 * wse) + align_up(8 * (size_t)k) +
                                     align_up(8 * qr_tblk_elems(mA, k)) + 4096));
    double *ws = take<double>(ctx, wse);
    double *tau = take<double>(ctx, k);
    double *Tb = take<double>(ctx, qr_tblk_elems(mA, k));
    FTT_CHECK(qr_factor(ctx, mA, k, Yk, mA, tau, Tb, ws, wse));
    FTT_CHECK(launch_identity(ctx, mA, k, st->Qk, mA));
    FTT_CHECK(qr_apply_q(ctx, mA, k, Yk, mA, Tb, k, st->Qk, mA, ws, wse));
    FTT_CHECK(project(k));
  }
  owned_free(ctx, Om);
  owned_free(ctx, Yk);
  owned_free(ctx, sk);
  owned_free(ctx, fro2_dev);
  *rest2_host = rest2;
  // Acceptance: the residual energy must sit below the rounding noise a
  // backward-stable full SVD already carries in the tail sums
  // (~ nA (eps ||A||_F)^2, the reference's own gesdd), or below 1e-8 delta^2,
  // and never above 1e-6 delta^2 (so tail(k) <= delta^2 and the rank <= k).
  const double eps = 2.220446049250313e-16;
  const double noise2 = (double)nA * eps * eps * fro2;
  const double thr = std::min(std::max(1e-8 * delta2, noise2), 1e-6 * delta2);
  static const bool debug = getenv("FTT_DEBUG") != nullptr;
  // strict (accepted = 2): the residual is below the noise of a full SVD's
  // tails; loose (accepted = 1): rest2 <= 1e-6 delta^2, usable when the
  // caller checks that its rank decision is the same at both ends of the
  // certified interval [tail_B, tail_B + rest2] (dense.py)
  const bool strict = rest2 <= thr, loose = rest2 <= 1e-6 * delta2;
  if (debug)
    fprintf(stderr, "[ftt] lowrank m=%lld n=%lld k=%lld rest2=%.3e thr=%.3e -> %s\n",
            (long long)m, (long long)n, (long long)k, rest2, thr,
            strict ? "accepted" : (loose ? "accepted (interval)" : "rejected"));
  if (!loose) return FTT_OK;  // (a speculative inner state is released with st)
  if (!st->inner) {
    st->inner = new SvdState();
    FTT_CHECK(svd_factor(ctx, st->inner, k, nA, st->Bk, k, 0, nullptr, nullptr, true));
  }
  st->sigma = st->inner->sigma;
  if (s_host) memcpy(s_host, st->sigma.data(), 8 * st->sigma.size());
  *accepted = strict ? 2 : 1;
  return FTT_OK;
}

extern "C" int ftt_svd_lowrank_f64(ftt_ctx *ctx, int64_t m, int64_t n, const double *A,
                                   int64_t lda, int32_t a_row_major, int64_t k, double delta2,
                                   double *s_host, double *rest2_host, int32_t *accepted) {
  return lowrank_run(ctx, m, n, A, lda, a_row_major, nullptr, k, delta2, s_host, rest2_host,
                     accepted);
}

static std::atomic<int64_t> g_scatter_steps{0};

int ftt::svd_lowrank_scatter(ftt_ctx *ctx, ScatterOperand *op, int64_t k, double delta2,
                             double *s_host, double *rest2_host, int32_t *accepted) {
  const int64_t m = op->r * op->n, n = op->mA;
  if (!ctx || !accepted || !rest2_host || m >= n || !scatter_operand_ok(op->mA, op->n, op->r, op->K)) {
    set_error("svd_lowrank_scatter: invalid operand");
    return FTT_ERR_INVALID;
  }
  *accepted = 0;
  *rest2_host = -1.0;
  FTT_CHECK(scatter_operand_build(ctx, op));
  const int rc = lowrank_run(ctx, m, n, nullptr, 0, 1, nullptr, k, delta2, s_host, rest2_host,
                             accepted, op);
  scatter_operand_free(ctx, op);
  if (rc == FTT_OK && *accepted) ++g_scatter_steps;
  return rc;
}

extern "C" int64_t ftt_scatter_steps(void) { return g_scatter_steps.load(); }

extern "C" int ftt_svd_lowrank_sparse_f64(ftt_ctx *ctx, int64_t m, int64_t n, int64_t nnz,
                                          const int64_t *fiber_of, const int64_t *pivot_index,
                                          const double *values, const int64_t *t_map,
                                          const int64_t *s_map, int64_t n_p, int64_t k,
                                          double delta2, double *s_host, double *rest2_host,
                                          int32_t *accepted) {
  if (!ctx || m < 1 || n < 1 || nnz < 1 || n_p < 1 || !fiber_of || !pivot_index || !values ||
      !accepted || !rest2_host) {
    set_error("ftt_svd_lowrank_sparse_f64: invalid arguments");
    return FTT_ERR_INVALID;
  }
  if (m > 0x7fffffffLL || n > 0x7fffffffLL || nnz >= ((int64_t)1 << 30)) {
    set_error("ftt_svd_lowrank_sparse_f64: operand too large for 32-bit entry indices");
    return FTT_ERR_INVALID;
  }
  return svd_lowrank_sparse(ctx, m, n, nnz, fiber_of, pivot_index, values, t_map, s_map, n_p, 0,
                            nullptr, k, delta2, s_host, rest2_host, accepted);
}

int ftt::svd_lowrank_sparse(ftt_ctx *ctx, int64_t m, int64_t n, int64_t nnz,
                            const int64_t *fiber_of, const int64_t *pivot_index,
                            const double *values, const int64_t *t_map, const int64_t *s_map,
                            int64_t n_p, int64_t R, const int64_t *indptr, int64_t k,
                            double delta2, double *s_host, double *rest2_host, int32_t *accepted) {
  *accepted = 0;
  *rest2_host = -1.0;
  SparseOperand op;
  FTT_CHECK(sparse_operand_build(ctx, &op, nnz, fiber_of, pivot_index, values, t_map, s_map, n_p, m,
                                 n, R, indptr));
  const int rc = lowrank_run(ctx, m, n, nullptr, 0, 1, &op, k, delta2, s_host, rest2_host, accepted);
  sparse_operand_free(ctx, &op);
  return rc;
}

extern "C" int ftt_svd_vectors(ftt_ctx *ctx, int64_t rank, double *U, int64_t ldu,
                               int32_t u_row_major, double *V, int64_t ldv, int32_t v_row_major,
                               int32_t scale_v) {
  if (!ctx || !ctx->svd) {
    set_error("ftt_svd_vectors: no factorization in this context");
    return FTT_ERR_INVALID;
  }
  SvdState *st = ctx->svd;
  const int64_t mA = st->mA, nA = st->nA;
  if (rank < 0 || rank > (int64_t)st->sigma.size()) {
    set_error("rank %lld out of range", (long long)rank);
    return FTT_ERR_INVALID;
  }
  if (rank == 0) return FTT_OK;
  double *UA = nullptr, *VA = nullptr, *UAi = nullptr, *VAi = nullptr, *sig2 = nullptr,
         *fac = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&UA, 8 * (size_t)mA * rank));
  if (st->lowrank) {
    // A_tall ~= Qk B with B = U_B S V_B^T  =>  U_A = Qk U_B, V_A = V_B (used
    // in place in the inner state's output, no copy)
    SvdState *in = st->inner;
    FTT_CHECK(owned_alloc(ctx, (void **)&UAi, 8 * (size_t)in->mA * rank));
    FTT_CHECK(owned_alloc(ctx, (void **)&VAi, 8 * (size_t)in->nA * rank));
    FTT_CHECK(svd_raw_vectors(ctx, in, rank, UAi, VAi, st->sigma.data(), &sig2));
    const int64_t k = in->m;  // B is k x nA
    double *UB = in->transposed ? VAi : UAi;  // k x rank
    VA = in->transposed ? UAi : VAi;          // nA x rank
    FTT_CHECK(gemm(ctx, 0, 0, mA, rank, k, 1.0, st->Qk, mA, UB, k, 0.0, UA, mA, nullptr, 0));
  } else {
    FTT_CHECK(owned_alloc(ctx, (void **)&VA, 8 * (size_t)nA * rank));
    FTT_CHECK(svd_raw_vectors(ctx, st, rank, UA, VA, st->sigma.data(), &sig2));
  }
  double *UM = st->transposed ? VA : UA;
  double *VM = st->transposed ? UA : VA;
  const int64_t mu = st->transposed ? nA : mA;  // == caller m
  const int64_t mv = st->transposed ? mA : nA;  // == caller n
  {
    // (sig2 was staged with the selection; the arena block stays valid: no
    // reservation happened since)
    fac = sig2 + rank;
    k_sign_pick<<<(unsigned)rank, 256, 0, ctx->stream>>>(mu, UM, mu, fac);
    FTT_LAUNCHED(ctx);
    if (rank <= 32) {
      // narrow factors: one fused pass (row-major reads stay within a few
      // sectors per warp)
      if (U || V) {
        const int64_t tot = (U ? mu * rank : 0) + (V ? mv * rank : 0);
        k_sign_write<<<grid_for(tot, 256, 4), 256, 0, ctx->stream>>>(
            mu, mv, rank, UM, VM, fac, sig2, scale_v, U, ldu, u_row_major, V, ldv, v_row_major);
        FTT_LAUNCHED(ctx);
      }
    } else {
      // wide factors: in-place sign pass, then tiled transposes / copies
      const int64_t nch =
          std::max<int64_t>(1, std::min<int64_t>(64, ceil_div(std::max(mu, mv), 4096)));
      k_sign_apply<<<dim3((unsigned)rank, (unsigned)nch), 256, 0, ctx->stream>>>(
          mu, mv, UM, mu, VM, mv, fac, sig2, scale_v);
      FTT_LAUNCHED(ctx);
      if (U) {
        if (u_row_major) FTT_CHECK(transpose(ctx, mu, rank, UM, mu, U, ldu));
        else FTT_CHECK(copy_matrix(ctx, mu, rank, UM, mu, U, ldu));
      }
      if (V) {
        if (v_row_major) FTT_CHECK(transpose(ctx, mv, rank, VM, mv, V, ldv));
        else FTT_CHECK(copy_matrix(ctx, mv, rank, VM, mv, V, ldv));
      }
    }
  }
  owned_free(ctx, UA);
  if (st->lowrank) {
    owned_free(ctx, UAi);
    owned_free(ctx, VAi);
  } else {
    owned_free(ctx, VA);
  }
  return FTT_OK;
}
