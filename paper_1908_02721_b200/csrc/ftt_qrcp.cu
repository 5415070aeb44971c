// Householder QR with column pivoting (LAPACK dgeqp3 semantics: the pivot is
// the remaining column of largest partial norm, ties to the lowest position)
// of the n x n triangular factor R of an SVD operand -- the preconditioner of
// the one-sided Jacobi SVD (Drmac-Veselic): A P = (Q Q2) R2 is a pivoted QR
// of A, and Jacobi on X = R2^T converges in fewer sweeps with fewer active
// pairs than on R^T.
//
// One cooperative launch; each CTA owns the physical columns c = b, b + G,
// ...; the column permutation is a logical -> physical map kept (identically)
// in every CTA's shared memory, so no column moves.  Per step j:
//   * every CTA reads the pivot column p (physical) rows j.. from global
//     memory and forms the reflector's scalars itself (same operands, same
//     order: bitwise the same in every CTA);
//   * each CTA updates its own remaining columns (a warp per column: dot,
//     axpy), downdates their partial norms (recomputed when the downdate
//     cancels, LAPACK's tol3z rule) and publishes its best candidate;
//   * one grid barrier; every CTA reads all candidates and picks the next
//     pivot; the owner of the previous pivot stores its reflector (scaled by
//     1/v0) and beta -- nobody reads that column any more.
// Output (logical order, after ftt_qrcp_gather): reflectors below the
// diagonal, R2 on and above it, tau, perm (logical -> original column).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "ftt_dense.cuh"

namespace ftt {
namespace {

namespace cg = cooperative_groups;

constexpr int QP_NT = 256;
constexpr int QP_MAXN = 8192;  // perm + inverse in shared memory (2 x 32 KB)

__device__ __forceinline__ double qp_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(QP_NT) k_qrcp(int n, double *__restrict__ B, int64_t ldb,
                                                double *__restrict__ tau,
                                                double *__restrict__ vn1,
                                                double *__restrict__ vn2,
                                                double *__restrict__ cand_v,
                                                int *__restrict__ cand_i,
                                                int *__restrict__ perm_out) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ int qp_sm[];
  int *perm = qp_sm;           // logical -> physical
  int *ipos = qp_sm + n;       // physical -> logical
  __shared__ double s_red[QP_NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = QP_NT / 32;
  const int G = gridDim.x, b = blockIdx.x;
  const double tol3z = sqrt(2.220446049250313e-16);
  for (int i = tid; i < n; i += QP_NT) {
    perm[i] = i;
    ipos[i] = i;
  }
  // initial column norms of the owned columns
  for (int c = b + G * warp; c < n; c += G * nw) {
    const double *col = B + (int64_t)c * ldb;
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += col[i] * col[i];
    s = qp_warp_sum(s);
    if (lane == 0) {
      vn1[c] = s;
      vn2[c] = s;
    }
  }
  __syncthreads();
  grid.sync();
  int prev = -1;  // physical column of the previous pivot
  double prev_v0 = 1.0, prev_beta = 0.0, prev_tau = 0.0;
  for (int j = 0; j < n; ++j) {
    // ---- pivot: largest partial norm among logical positions >= j
    int p;
    if (j == 0) {
      // every CTA scans all norms (written before the barrier above)
      double bv = -1.0;
      int bi = -1;
      for (int c = tid; c < n; c += QP_NT) {
        const double v = vn1[c];
        if (v > bv || (v == bv && c < bi)) {
          bv = v;
          bi = c;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi >= 0 && (bi < 0 || oi < bi))) {
          bv = ov;
          bi = oi;
        }
      }
      __shared__ double s_bv[QP_NT / 32];
      __shared__ int s_bi[QP_NT / 32];
      if (lane == 0) {
        s_bv[warp] = bv;
        s_bi[warp] = bi;
      }
      __syncthreads();
      double best = -1.0;
      int bidx = -1;
      for (int w = 0; w < nw; ++w)
        if (s_bv[w] > best || (s_bv[w] == best && s_bi[w] >= 0 && s_bi[w] < bidx)) {
          best = s_bv[w];
          bidx = s_bi[w];
        }
      p = bidx;
    } else {
      // the CTAs' candidates, one per thread (G <= QP_NT), block arg-max
      // (largest norm, ties to the lowest logical position)
      double bv = -1.0;
      int bpos = n;
      for (int g = tid; g < G; g += QP_NT) {
        const int c = cand_i[g];
        if (c < 0) continue;
        const double v = cand_v[g];
        const int pos = ipos[c];
        if (v > bv || (v == bv && pos < bpos)) {
          bv = v;
          bpos = pos;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int op = __shfl_xor_sync(0xffffffffu, bpos, o);
        if (ov > bv || (ov == bv && op < bpos)) {
          bv = ov;
          bpos = op;
        }
      }
      __shared__ double s_pv[QP_NT / 32];
      __shared__ int s_pp[QP_NT / 32];
      if (lane == 0) {
        s_pv[warp] = bv;
        s_pp[warp] = bpos;
      }
      __syncthreads();
      double best = -1.0;
      int pbest = n;
      for (int w = 0; w < nw; ++w)
        if (s_pv[w] > best || (s_pv[w] == best && s_pp[w] < pbest)) {
          best = s_pv[w];
          pbest = s_pp[w];
        }
      p = perm[pbest];
    }
    __syncthreads();
    // swap logical positions j and ipos[p] (every CTA, identically)
    if (tid == 0) {
      const int pj = perm[j], pp = ipos[p];
      perm[pp] = pj;
      ipos[pj] = pp;
      perm[j] = p;
      ipos[p] = j;
    }
    // the previous pivot's owner stores its reflector and beta
    if (prev >= 0 && prev % G == b) {
      double *col = B + (int64_t)prev * ldb;
      const double inv = 1.0 / prev_v0;
      if (prev_tau != 0.0)
        for (int i = j + tid; i < n; i += QP_NT) col[i] *= inv;
      if (tid == 0) {
        col[j - 1] = prev_beta;
        tau[j - 1] = prev_tau;
      }
    }
    __syncthreads();
    // ---- reflector scalars from the pivot column (rows j..), in every CTA
    const double *pc = B + (int64_t)p * ldb;
    double sub = 0.0;
    for (int i = j + 1 + tid; i < n; i += QP_NT) sub += pc[i] * pc[i];
    sub = qp_warp_sum(sub);
    if (lane == 0) s_red[warp] = sub;
    __syncthreads();
    sub = 0.0;
    for (int w = 0; w < nw; ++w) sub += s_red[w];
    const double alpha = pc[j];
    double tj = 0.0, beta = alpha, v0 = 1.0;
    if (sub > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + sub), alpha);
      v0 = alpha - beta;
      tj = (beta - alpha) / beta;
    }
    const double inv0 = 1.0 / v0;
    // ---- update the owned remaining columns (a warp each)
    double best = -1.0;
    int bcol = -1;
    for (int c = b + G * warp; c < n; c += G * nw) {
      if (ipos[c] <= j) continue;  // processed (or the pivot)
      double *col = B + (int64_t)c * ldb;
      if (tj != 0.0) {
        double d = 0.0;
        for (int i = j + 1 + lane; i < n; i += 32) d += pc[i] * col[i];
        d = qp_warp_sum(d);
        const double w = tj * (col[j] + d * inv0);
        for (int i = j + 1 + lane; i < n; i += 32) col[i] -= w * (pc[i] * inv0);
        __syncwarp();
        if (lane == 0) col[j] -= w;
        __syncwarp();
      }
      // partial norm of rows j+1.. (dgeqp3's downdate, recomputed on cancellation)
      double nv = 0.0;
      if (lane == 0) {
        const double r = col[j];
        double v1 = vn1[c];
        if (v1 != 0.0) {
          double temp = 1.0 - (r * r) / v1;
          temp = temp < 0.0 ? 0.0 : temp;
          const double temp2 = temp * (v1 / vn2[c]);
          nv = temp2 <= tol3z ? -1.0 : v1 * temp;  // -1: recompute
        }
      }
      nv = __shfl_sync(0xffffffffu, nv, 0);
      if (nv < 0.0) {
        double s = 0.0;
        for (int i = j + 1 + lane; i < n; i += 32) s += col[i] * col[i];
        s = qp_warp_sum(s);
        nv = s;
        if (lane == 0) vn2[c] = s;
      }
      if (lane == 0) vn1[c] = nv;
      if (nv > best || (nv == best && (bcol < 0 || ipos[c] < ipos[bcol]))) {
        best = nv;
        bcol = c;
      }
    }
    // CTA candidate: best over warps (ties -> lowest logical position)
    __shared__ double s_cv[QP_NT / 32];
    __shared__ int s_ci[QP_NT / 32];
    if (lane == 0) {
      s_cv[warp] = best;
      s_ci[warp] = bcol;
    }
    __syncthreads();
    if (tid == 0) {
      double bv = -1.0;
      int bi = -1;
      for (int w = 0; w < nw; ++w) {
        const int c = s_ci[w];
        if (c < 0) continue;
        if (s_cv[w] > bv || (s_cv[w] == bv && ipos[c] < ipos[bi])) {
          bv = s_cv[w];
          bi = c;
        }
      }
      cand_v[b] = bv;
      cand_i[b] = bi;
    }
    prev = p;
    prev_v0 = v0;
    prev_beta = beta;
    prev_tau = tj;
    __syncthreads();
    grid.sync();
  }
  // the last pivot's reflector (its tail is empty: tau = 0) and the map
  if (prev >= 0 && prev % G == b && threadIdx.x == 0) {
    B[(int64_t)prev * ldb + (n - 1)] = prev_beta;
    tau[n - 1] = prev_tau;
  }
  if (b == 0)
    for (int i = tid; i < n; i += QP_NT) perm_out[i] = perm[i];
}

// Out[:, j] = B[:, perm[j]] (logical column order).
__global__ void k_gather_perm_cols(int n, const double *__restrict__ B, int64_t ldb,
                                   const int *__restrict__ perm, double *__restrict__ Out,
                                   int64_t ldo) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / n), i = (int)(e - (int64_t)j * n);
    Out[i + (int64_t)j * ldo] = B[i + (int64_t)perm[j] * ldb];
  }
}

}  // namespace

bool qrcp_ok(int64_t n) { return n >= 2 && n <= QP_MAXN; }

// B (n x n, ld n) -> Out (n x n, ld n): reflectors below the diagonal, R2 on
// and above it (logical order), tau (n), perm (n: logical -> original
// column).  Scratch: 2 n doubles + a few per CTA.
int qrcp_factor(ftt_ctx *ctx, int64_t n64, double *B, double *Out, double *tau, int *perm) {
  const int n = (int)n64;
  if (!qrcp_ok(n64)) {
    set_error("qrcp_factor: n out of range");
    return FTT_ERR_INVALID;
  }
  const size_t smem = 2 * sizeof(int) * (size_t)n;
  static bool attr = false;
  if (!attr) {
    FTT_CUDA(cudaFuncSetAttribute(k_qrcp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(2 * sizeof(int) * QP_MAXN)));
    attr = true;
  }
  int per_sm = 0;
  FTT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_qrcp, QP_NT, smem));
  // one CTA per SM at most (every step reads the pivot column in each CTA);
  // few columns per CTA keeps the warps busy
  int G = std::min<int>(ctx->num_sms * std::max(1, std::min(per_sm, 1)),
                        std::max<int>(1, (int)ceil_div(n, 8)));
  double *scratch = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&scratch, sizeof(double) * (2 * (size_t)n + 2 * (size_t)G)));
  double *vn1 = scratch, *vn2 = scratch + n, *cv = scratch + 2 * (size_t)n;
  int *ci = reinterpret_cast<int *>(cv + G);
  int ldb = n;
  int64_t ldb64 = ldb;
  void *args[] = {(void *)&n, &B, &ldb64, &tau, &vn1, &vn2, &cv, &ci, &perm};
  const int pb = prof_begin(ctx);
  FTT_CUDA(cudaLaunchCooperativeKernel((const void *)k_qrcp, dim3(G), dim3(QP_NT), args, smem,
                                       ctx->stream));
  FTT_LAUNCHED(ctx);
  k_gather_perm_cols<<<grid_for((int64_t)n * n, 256, 4), 256, 0, ctx->stream>>>(n, B, n, perm, Out, n);
  FTT_LAUNCHED(ctx);
  // (4/3) n^3 flops; the trailing matrix read and written once per step
  prof_end(ctx, pb, PT_QR_PANEL, 16.0 * (double)n * n * n / 3.0, 4.0 * (double)n * n * n / 3.0);
  owned_free(ctx, scratch);
  return FTT_OK;
}

}  // namespace ftt
