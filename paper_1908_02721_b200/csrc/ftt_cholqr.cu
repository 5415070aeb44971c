// Numerical rank and a spanning column subset of the low-rank sketch
// Y = A Omega (mA x k, k <= 64) from its Gram matrix:
//
//   G = Y^T Y                     (DMMA GEMM, split-K over the mA rows)
//   G = P L L^T P^T, stop at the first pivot <= tau * max diag(G)
//       -> rank r, pivot order P   (one CTA)
//
// The caller then factors only the r selected columns with the Householder
// TSQR (ftt_small.cu): the low-rank sketches of the BASELINE configs have
// k = 2 r + 8 columns, so the column-sequential QR shrinks from k to r
// steps.  (Using Q = Y_sel L11^-T directly -- CholeskyQR2 -- was measured to
// lose ~30x in the residual certificate: the GEMM with L11^-T carries
// eps * cond(Y_sel) subspace error.)  Dropping sketch directions below
// sqrt(tau) of the largest is safe because the caller certifies the basis
// with the explicit residual ||A - Q Q^T A||_F and takes the full SVD when
// the certificate fails.
#include <algorithm>
#include <cmath>
#include <vector>

#include "ftt_dense.cuh"

namespace ftt {
namespace {

constexpr int CQ_MAX = 64;

// Pivoted Cholesky of the k x k SPD-ish G (ld ldg): G = P L L^T P^T, stopping
// at the first pivot <= tau * max diag(G).  out[0] = r, piv_out[0..k) = P
// (the first r entries are a well-conditioned spanning column subset).
// The matrix is never permuted: it stays in the original index order, a
// `done` mask marks eliminated indices and the Schur complement is updated
// in place on the rest.  One CTA of CQ_NT threads, thread t owns row t % 64
// and columns t / 64 + 8 q of the update (no integer division); warp 0 picks
// the pivot by a shuffle argmax (largest diagonal, lowest index on ties).
// Three barriers per step.
constexpr int CQ_NT = 512;
__global__ void __launch_bounds__(CQ_NT) k_chol_inv(int k, const double *__restrict__ G, int64_t ldg,
                                                    double tau, int *__restrict__ out,
                                                    int64_t *__restrict__ piv_out,
                                                    const double *__restrict__ aux_src,
                                                    double *__restrict__ aux_dst) {
  extern __shared__ double cq_smem[];
  double(*A)[CQ_MAX + 1] = reinterpret_cast<double(*)[CQ_MAX + 1]>(cq_smem);  // Schur complement
  __shared__ double lcol[CQ_MAX];
  __shared__ int done[CQ_MAX];
  __shared__ int order[CQ_MAX];
  __shared__ double dmax0;
  __shared__ int s_p, s_stop;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int e = tid; e < k * k; e += blockDim.x) {
    const int i = e % k, j = e / k;
    // symmetrise (the two triangles of a GEMM Gram may differ in the last bit)
    A[i][j] = 0.5 * (G[i + (int64_t)j * ldg] + G[j + (int64_t)i * ldg]);
  }
  if (tid < k) done[tid] = 0;
  if (tid == 0 && aux_src) *aux_dst = *aux_src;  // caller's scalar rides on the rank read
  __syncthreads();
  if (tid < 32) {
    double m = 0.0;
    for (int i = lane; i < k; i += 32) m = fmax(m, A[i][i]);
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) dmax0 = m;
  }
  const int ra = tid & (CQ_MAX - 1), cb0 = tid / CQ_MAX;
  constexpr int CSTEP = CQ_NT / CQ_MAX;
  int r = k;
  for (int j = 0; j < k; ++j) {
    __syncthreads();  // previous update (and dmax0) visible
    if (tid < 32) {
      double best = -INFINITY;
      int p = k;
      for (int i = lane; i < k; i += 32)
        if (!done[i] && (A[i][i] > best || p == k)) {
          best = A[i][i];
          p = i;
        }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int op = __shfl_xor_sync(0xffffffffu, p, o);
        if (op < k && (p == k || ob > best || (ob == best && op < p))) {
          best = ob;
          p = op;
        }
      }
      if (lane == 0) {
        s_p = p;
        s_stop = !(best > fmax(tau, 0.0) * dmax0) || !(best > 0.0);
        if (!s_stop) {
          order[j] = p;
          done[p] = 1;
        }
      }
    }
    __syncthreads();
    if (s_stop) {
      r = j;
      break;
    }
    const int p = s_p;
    if (tid < k) {
      const double ljj = sqrt(A[p][p]);
      lcol[tid] = done[tid] ? 0.0 : A[tid][p] / ljj;
    }
    __syncthreads();
    if (ra < k && !done[ra]) {
      const double la = lcol[ra];
      for (int b = cb0; b < k; b += CSTEP) A[ra][b] -= la * lcol[b];
    }
  }
  __syncthreads();
  if (piv_out && tid < k) {
    // pivots in elimination order, then the never-chosen indices ascending
    if (tid < r) piv_out[tid] = order[tid];
    if (!done[tid]) {
      int pos = r;
      for (int i = 0; i < tid; ++i) pos += !done[i];
      piv_out[pos] = tid;
    }
  }
  if (tid == 0) out[0] = r;
}

constexpr size_t CQ_SMEM = sizeof(double) * CQ_MAX * (CQ_MAX + 1);

}  // namespace

// Numerical rank r of the sketch Y (mA x k, ld mA) from a pivoted Cholesky
// of Y^T Y (relative pivot cutoff tau) and the pivot order (sel_dev[0..r)
// are the columns of a well-conditioned spanning subset).
// The same factorisation without the host round trip: the rank word lands in
// *rank_dev (a device int the caller reads back later with other results).
int sketch_rank_async(ftt_ctx *ctx, int64_t mA, int64_t k, const double *Y, double tau,
                      int64_t *sel_dev, int *rank_dev) {
  if (k <= 0 || k > CQ_MAX) {
    set_error("sketch_rank: k out of range");
    return FTT_ERR_INVALID;
  }
  static bool attr = false;
  if (!attr) {
    FTT_CUDA(cudaFuncSetAttribute(k_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)CQ_SMEM));
    attr = true;
  }
  const size_t ske = std::max(gemm_splitk_elems(k, k, mA), (size_t)1);
  double *blk = nullptr;  // G (k x k) | split-K space
  FTT_CHECK(owned_alloc(ctx, (void **)&blk, 8 * ((size_t)k * k + ske)));
  double *G = blk, *sk = G + (size_t)k * k;
  FTT_CHECK(gemm(ctx, 1, 0, k, k, mA, 1.0, Y, mA, Y, mA, 0.0, G, k, sk, ske));
  k_chol_inv<<<1, CQ_NT, CQ_SMEM, ctx->stream>>>((int)k, G, k, tau, rank_dev, sel_dev, nullptr,
                                                 nullptr);
  FTT_LAUNCHED(ctx);
  owned_free(ctx, blk);
  return FTT_OK;
}

int sketch_rank(ftt_ctx *ctx, int64_t mA, int64_t k, const double *Y, double tau, int64_t *sel_dev,
                int64_t *rank, const double *aux_dev, double *aux_host) {
  *rank = 0;
  if (k <= 0 || k > CQ_MAX) {
    set_error("sketch_rank: k out of range");
    return FTT_ERR_INVALID;
  }
  static bool attr = false;
  if (!attr) {
    FTT_CUDA(cudaFuncSetAttribute(k_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)CQ_SMEM));
    attr = true;
  }
  const size_t ske = std::max(gemm_splitk_elems(k, k, mA), (size_t)1);
  // one allocation: rank word + aux scalar (16 B) | G (k x k) | split-K space
  double *blk = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&blk, 8 * (2 + (size_t)k * k + ske)));
  int *dev_r = reinterpret_cast<int *>(blk);
  double *G = blk + 2, *sk = G + (size_t)k * k;
  FTT_CHECK(gemm(ctx, 1, 0, k, k, mA, 1.0, Y, mA, Y, mA, 0.0, G, k, sk, ske));
  // one round trip for the rank and the caller's device scalar (copied by
  // the kernel)
  k_chol_inv<<<1, CQ_NT, CQ_SMEM, ctx->stream>>>((int)k, G, k, tau, dev_r, sel_dev, aux_dev, blk + 1);
  FTT_LAUNCHED(ctx);
  int hb[4] = {0, 0, 0, 0};
  FTT_CHECK(copy_to_host(ctx, hb, dev_r, aux_dev ? 16 : 4));
  const int r = hb[0];
  if (aux_dev && aux_host) memcpy(aux_host, hb + 2, sizeof(double));
  owned_free(ctx, blk);
  *rank = r;
  return FTT_OK;
}

}  // namespace ftt
