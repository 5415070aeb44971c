// Internal dense fp64 building blocks shared by the QR / SVD / TT files.
#pragma once
#include "ftt_common.cuh"

namespace ftt {

// Column-major DMMA GEMM (see ftt_gemm.cu).  splitk_ws may be NULL (no
// split-K); otherwise it must hold gemm_splitk_elems(m, n, k) doubles.
int gemm(ftt_ctx *ctx, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha,
         const double *A, int64_t lda, const double *B, int64_t ldb, double beta, double *C,
         int64_t ldc, double *splitk_ws, size_t splitk_ws_elems);
size_t gemm_splitk_elems(int64_t m, int64_t n, int64_t k);
// ||R0 - op(A) op(B)||_F^2 without materialising the residual (R0 stored
// transposed when r_trans), to the host (out_host) and/or left in device
// memory (out_dev).
int gemm_resid_sumsq(ftt_ctx *ctx, int ta, int tb, int64_t m, int64_t n, int64_t k,
                     const double *A, int64_t lda, const double *B, int64_t ldb, const double *R0,
                     int64_t ldr, int r_trans, double *out_host, double *out_dev = nullptr);
int transpose(ftt_ctx *ctx, int64_t rows, int64_t cols, const double *src, int64_t lds,
              double *dst, int64_t ldd);

// Blocked Householder QR (ftt_qr.cu).  Factors the m x n column-major A in
// place (LAPACK dgeqrf layout: R on and above the diagonal, reflectors
// below, tau[min(m,n)]) and stores the block T factors (NBO x NBO each) in
// Tblk.  Workspace sizes from qr_workspace_elems.
constexpr int QR_NBO = 128;  // outer block (trailing update)
constexpr int QR_NBI = 32;   // inner panel (cooperative column-by-column)
size_t qr_workspace_elems(int64_t m, int64_t n);
size_t qr_tblk_elems(int64_t m, int64_t n);
int qr_factor(ftt_ctx *ctx, int64_t m, int64_t n, double *A, int64_t lda, double *tau,
              double *Tblk, double *ws, size_t ws_elems);
// Z (m x r, ldz) <- Q * Z using the factorization above (Q = H_1 ... H_k).
int qr_apply_q(ftt_ctx *ctx, int64_t m, int64_t n, const double *A, int64_t lda, const double *Tblk,
               int64_t r, double *Z, int64_t ldz, double *ws, size_t ws_elems);
size_t qr_apply_workspace_elems(int64_t m, int64_t n, int64_t r);
// The block T factors of an already factored A (reflectors below the
// diagonal, tau) in qr_factor's layout, so that qr_apply_q can use them.
int qr_build_tblk(ftt_ctx *ctx, int64_t m, int64_t n, const double *A, int64_t lda,
                  const double *tau, double *Tblk, double *ws, size_t ws_elems);

// Householder QR with column pivoting of an n x n matrix (ftt_qrcp.cu): B is
// overwritten (scratch); Out (n x n, ld n) gets the reflectors below the
// diagonal and R2 on and above it in pivoted order, tau (n), perm (n device
// ints: pivoted position -> original column).
bool qrcp_ok(int64_t n);
int qrcp_factor(ftt_ctx *ctx, int64_t n, double *B, double *Out, double *tau, int *perm);

// Numerical rank r of the sketch Y (mA x k <= 64) and its pivot order
// (sel_dev, k entries; the first r span Y) from a pivoted Cholesky of the
// Gram (ftt_cholqr.cu).
// aux_dev (optional): one device double fetched in the same round trip.
int sketch_rank(ftt_ctx *ctx, int64_t mA, int64_t k, const double *Y, double tau, int64_t *sel_dev,
                int64_t *rank, const double *aux_dev = nullptr, double *aux_host = nullptr);

// Without the round trip: the rank word goes to *rank_dev (device).
int sketch_rank_async(ftt_ctx *ctx, int64_t mA, int64_t k, const double *Y, double tau,
                      int64_t *sel_dev, int *rank_dev);

// Sparse operand of the first truncation step (ftt_sparse.cu): the entries
// of the pivot core as A_tall (mA x nA = M or M^T) in CSR (by row) and CSC
// (by column, rows ascending) order.
struct SparseOperand {
  int64_t nnz = 0, mA = 0, nA = 0;
  bool transposed = false;
  int64_t *rptr = nullptr;   // mA + 1
  int32_t *cidx_r = nullptr; // CSR column per entry
  double *v_r = nullptr;     // CSR values
  int64_t *cptr = nullptr;   // nA + 1
  uint64_t *keyc = nullptr;  // CSC keys: the column (sorted, rows ascending within)
  int32_t *ridx_c = nullptr; // CSC row per entry
  int32_t *cidx_c = nullptr; // CSC column per entry
  double *v_c = nullptr;     // CSC values
  int64_t *seg_base = nullptr;  // nA + 1: first B segment of each column
  int64_t max_segs = 0;
  double *Qr = nullptr;      // row-major copy of the range basis (sparse_qt_a)
  int64_t ldq = 0;           // its row stride (kr rounded up to even)
  // fiber-level CSR (transposed operand with the fiber structure at hand):
  // rptr indexes fperm (fibers by row, ascending); no cidx_r / v_r
  bool by_fiber = false;
  uint32_t *fperm = nullptr;
  int64_t *fe0 = nullptr;   // sorted fiber j: first entry,
  int32_t *flen = nullptr;  // entry count,
  int32_t *fcb = nullptr;   // first column of its block (t_map * n_p)
  const int64_t *f_indptr = nullptr, *f_pidx = nullptr, *f_tmap = nullptr;
  const double *f_vals = nullptr;
  int64_t f_np = 0;
};
// M (m x n): entry e at row t_map[f] * np + pidx[e], column s_map[f]
// (f = fiber_of[e]; a NULL map means 0).
int sparse_operand_build(ftt_ctx *ctx, SparseOperand *op, int64_t nnz, const int64_t *fiber_of,
                         const int64_t *pidx, const double *vals, const int64_t *tmap,
                         const int64_t *smap, int64_t np, int64_t m, int64_t n, int64_t R = 0,
                         const int64_t *indptr = nullptr);
// ftt_svd_lowrank_sparse_f64 with the fiber structure (R fibers, indptr) for
// the fiber-level CSR (ftt_svd.cu).
int svd_lowrank_sparse(ftt_ctx *ctx, int64_t m, int64_t n, int64_t nnz, const int64_t *fiber_of,
                       const int64_t *pivot_index, const double *values, const int64_t *t_map,
                       const int64_t *s_map, int64_t n_p, int64_t R, const int64_t *indptr,
                       int64_t k, double delta2, double *s_host, double *rest2_host,
                       int32_t *accepted);
void sparse_operand_free(ftt_ctx *ctx, SparseOperand *op);
// Y (mA x k col-major) = A_tall Omega with the range finder's test matrix.
int sparse_sketch(ftt_ctx *ctx, const SparseOperand &op, int64_t k, double *Y);
// B (kr x nA col-major) = Q^T A_tall, Q mA x kr col-major.
int sparse_qt_a(ftt_ctx *ctx, SparseOperand &op, int64_t kr, const double *Q, double *B);
// ||A_tall - Q B||_F^2 over every element (deterministic) -> out_dev.
// (after sparse_qt_a with the same Q)
int sparse_resid(ftt_ctx *ctx, SparseOperand &op, int64_t kr, const double *Q, const double *B,
                 double *out_dev);

// Scattered operand of a right-sweep step (ftt_scatter.cu): carry V (K x r,
// col-major, ld ldv) times a 0/1 core given by its kept rows (K ascending
// values i * mA + c'), as A_tall (mA x r n): A_tall[c', a n + i] = V[c, a].
struct ScatterOperand {
  int64_t mA = 0, n = 0, r = 0, K = 0;
  const int64_t *kept = nullptr;
  const double *V = nullptr;
  int64_t ldv = 0;
  int32_t *pos = nullptr;   // n x mA: entry at (i, c') or -1 (scatter_operand_build)
  int64_t *iptr = nullptr;  // n + 1: first entry of each block column
};
bool scatter_operand_ok(int64_t mA, int64_t n, int64_t r, int64_t K);
int scatter_operand_build(ftt_ctx *ctx, ScatterOperand *op);
void scatter_operand_free(ftt_ctx *ctx, ScatterOperand *op);
int scatter_sketch(ftt_ctx *ctx, const ScatterOperand &op, int64_t k, double *Y);
int scatter_qt_a(ftt_ctx *ctx, const ScatterOperand &op, int64_t kr, const double *Q, double *B);
int scatter_resid(ftt_ctx *ctx, const ScatterOperand &op, int64_t kr, const double *Q,
                  const double *B, double *out_dev);
// The certified low-rank path (ftt_svd.cu) on a scattered operand: M is
// (r n) x mA row-major, m = r n < mA; same outputs as ftt_svd_lowrank_f64.
int svd_lowrank_scatter(ftt_ctx *ctx, ScatterOperand *op, int64_t k, double delta2, double *s_host,
                        double *rest2_host, int32_t *accepted);

int check_finite(ftt_ctx *ctx, int64_t m, int64_t n, const double *A, int64_t lda, bool *ok);
int copy_matrix(ftt_ctx *ctx, int64_t m, int64_t n, const double *src, int64_t lds, double *dst,
                int64_t ldd);

}  // namespace ftt
