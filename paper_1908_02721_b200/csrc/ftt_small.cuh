// Narrow (n <= 64) QR / SVD without grid barriers (ftt_small.cu).
#pragma once
#include "ftt_common.cuh"

namespace ftt {

// A_tall (M x n) is `A` column-major (ld lda) or its transpose (trans).
bool tsqr_ok(int64_t m, int64_t n);

// Q (M x n, ld ldq) and R (n x n, ld ldr, diag >= 0; may be NULL) of A_tall.
// check = false skips the finite-input check (no host round trip) when the
// caller already knows the input is finite.
int tsqr_q(ftt_ctx *ctx, int64_t M, int64_t n, const double *A, int64_t lda, int trans, double *Q,
           int64_t ldq, double *R, int64_t ldr, bool check = true);

// Thin SVD core: U = Q P (M x n, ld ldu), Y = R^T P (n x n), norms_host[j] =
// ||Y_j|| (unsorted; sigma up to the caller's permutation).  One host round
// trip, which also brings back the caller's device scalar extra_dev (if any)
// into *extra_host (extra_n consecutive doubles, 1 <= extra_n <= 4).
int tsqr_svd(ftt_ctx *ctx, int64_t M, int64_t n, const double *A, int64_t lda, int trans, double *U,
             int64_t ldu, double *Y, double *norms_host, int *sweeps,
             const double *extra_dev = nullptr, double *extra_host = nullptr, int extra_n = 1);

// Short tall operands (n <= 16, A_tall and its reflectors fit in shared
// memory): the tsqr_svd factorisation in one CTA (k_jacobi_qr).  U = Q P
// (m x n), Yt = R^T P (n x n), norms_host = ||Yt_j|| unsorted.
bool direct_small_ok(int64_t m, int64_t n);
int direct_small_svd(ftt_ctx *ctx, int64_t m, int64_t n, const double *A, int64_t lda, int trans,
                     double *U, double *Yt, double *norms_host, int *sweeps,
                     const double *extra_dev = nullptr, double *extra_host = nullptr,
                     int extra_n = 1);

}  // namespace ftt
