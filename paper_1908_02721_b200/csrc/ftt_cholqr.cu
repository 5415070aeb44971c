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

// Pivoted (or plain, tau < 0) Cholesky of the k x k SPD-ish G (ld ldg) and
// M = P[:, :r] L11^-T written to M (k x k, ld k; columns >= r zero).
// out[0] = r.  One CTA of 256 threads.
__global__ void __launch_bounds__(256) k_chol_inv(int k, const double *__restrict__ G, int64_t ldg,
                                                  double tau, double *__restrict__ M,
                                                  int *__restrict__ out,
                                                  int64_t *__restrict__ piv_out) {
  extern __shared__ double cq_smem[];
  double(*A)[CQ_MAX + 1] = reinterpret_cast<double(*)[CQ_MAX + 1]>(cq_smem);  // working copy
  double(*L)[CQ_MAX + 1] = A + CQ_MAX;
  double(*R)[CQ_MAX + 1] = L + CQ_MAX;  // L11^-T = (L11^T)^-1, upper
  __shared__ int piv[CQ_MAX];
  __shared__ double dmax0;
  __shared__ int s_p, s_stop;
  const int tid = threadIdx.x;
  for (int e = tid; e < k * k; e += blockDim.x) {
    const int i = e % k, j = e / k;
    // symmetrise (the two triangles of a GEMM Gram may differ in the last bit)
    A[i][j] = 0.5 * (G[i + (int64_t)j * ldg] + G[j + (int64_t)i * ldg]);
    L[i][j] = 0.0;
  }
  if (tid < k) piv[tid] = tid;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < k; ++i) m = fmax(m, A[i][i]);
    dmax0 = m;
  }
  __syncthreads();
  int r = k;
  for (int j = 0; j < k; ++j) {
    if (tid == 0) {
      int p = j;
      if (tau >= 0.0) {
        double best = A[j][j];
        for (int i = j + 1; i < k; ++i)
          if (A[i][i] > best) {
            best = A[i][i];
            p = i;
          }
      }
      s_p = p;
      s_stop = !(A[p][p] > fmax(tau, 0.0) * dmax0) || !(A[p][p] > 0.0);
    }
    __syncthreads();
    if (s_stop) {
      r = j;
      break;
    }
    const int p = s_p;
    if (p != j) {  // symmetric swap of rows/cols j and p of A, rows of L, piv
      for (int t = tid; t < k; t += blockDim.x) {
        const double a = A[j][t];
        A[j][t] = A[p][t];
        A[p][t] = a;
      }
      __syncthreads();
      for (int t = tid; t < k; t += blockDim.x) {
        const double a = A[t][j];
        A[t][j] = A[t][p];
        A[t][p] = a;
        if (t < j) {
          const double l = L[j][t];
          L[j][t] = L[p][t];
          L[p][t] = l;
        }
      }
      if (tid == 0) {
        const int x = piv[j];
        piv[j] = piv[p];
        piv[p] = x;
      }
      __syncthreads();
    }
    // right-looking: A (trailing) holds the Schur complement
    const double ljj = sqrt(A[j][j]);
    for (int i = j + tid; i < k; i += blockDim.x) L[i][j] = i == j ? ljj : A[i][j] / ljj;
    __syncthreads();
    for (int e = tid; e < (k - j - 1) * (k - j - 1); e += blockDim.x) {
      const int a = j + 1 + e % (k - j - 1), b = j + 1 + e / (k - j - 1);
      A[a][b] -= L[a][j] * L[b][j];
    }
    __syncthreads();
  }
  // R = (L11^T)^-1 (upper, r x r): column c solves L11^T x = e_c backwards
  for (int c = tid; c < r; c += blockDim.x) {
    for (int i = r - 1; i >= 0; --i) {
      double s = i == c ? 1.0 : 0.0;
      for (int t = i + 1; t <= c; ++t) s -= L[t][i] * R[t][c];
      R[i][c] = i > c ? 0.0 : s / L[i][i];
    }
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += blockDim.x) {
    const int i = e % k, c = e / k;  // row i of the permuted order, column c
    M[piv[i] + (int64_t)c * k] = (i < r && c < r) ? R[i][c] : 0.0;
  }
  if (piv_out)
    for (int i = tid; i < k; i += blockDim.x) piv_out[i] = piv[i];
  if (tid == 0) out[0] = r;
}

constexpr size_t CQ_SMEM = 3 * sizeof(double) * CQ_MAX * (CQ_MAX + 1);

}  // namespace

// Numerical rank r of the sketch Y (mA x k, ld mA) from a pivoted Cholesky
// of Y^T Y (relative pivot cutoff tau) and the pivot order (sel_dev[0..r)
// are the columns of a well-conditioned spanning subset).
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
  double *G = nullptr, *M = nullptr, *sk = nullptr;
  int *dev_r = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&G, 8 * (size_t)k * k));
  FTT_CHECK(owned_alloc(ctx, (void **)&M, 8 * (size_t)k * k));
  FTT_CHECK(owned_alloc(ctx, (void **)&sk, 8 * ske));
  FTT_CHECK(owned_alloc(ctx, (void **)&dev_r, 64));
  FTT_CHECK(gemm(ctx, 1, 0, k, k, mA, 1.0, Y, mA, Y, mA, 0.0, G, k, sk, ske));
  k_chol_inv<<<1, 256, CQ_SMEM, ctx->stream>>>((int)k, G, k, tau, M, dev_r, sel_dev);
  FTT_LAUNCHED(ctx);
  // one round trip for the rank and the caller's device scalar
  if (aux_dev)
    FTT_CUDA(cudaMemcpyAsync(dev_r + 2, aux_dev, sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
  int hb[4] = {0, 0, 0, 0};
  FTT_CHECK(copy_to_host(ctx, hb, dev_r, aux_dev ? 16 : 4));
  const int r = hb[0];
  if (aux_dev && aux_host) memcpy(aux_host, hb + 2, sizeof(double));
  owned_free(ctx, G);
  owned_free(ctx, M);
  owned_free(ctx, sk);
  owned_free(ctx, dev_r);
  *rank = r;
  return FTT_OK;
}

}  // namespace ftt
