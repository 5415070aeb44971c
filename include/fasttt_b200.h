/*
 * fasttt_b200.h -- C ABI of the B200-native FastTT decomposition path.
 *
 * The reference (`sparsett`, pure Python, /root/reference/pkg/src/sparsett)
 * has no FFI; its boundary is the Python namespace.  Each entry point below
 * replaces the numpy/LAPACK body of one reference function on the hot path
 * (file:line cited per function).  The Python mirror of the reference API
 * (paper_1908_02721_b200/) binds these through ctypes.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers unless the name ends in `_host`.
 *  - Dense matrices are column-major with an explicit leading dimension
 *    (LAPACK convention); a row-major (numpy C-order) r x c array is the
 *    column-major c x r array of its transpose.
 *  - Sizes are int64_t; every call is enqueued on the context's stream.
 *    Calls that return a size to the host (`*_out` host pointers)
 *    synchronise that stream.
 *  - Return value: FTT_OK or an ftt_status error; ftt_last_error() gives a
 *    message.  No exception crosses the ABI.
 *  - Workspaces are owned by the context (grow-only, stream-ordered).
 */
#ifndef FASTTT_B200_H
#define FASTTT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FTT_OK = 0,
  FTT_ERR_INVALID = 1,   /* -> ValueError / TypeError in the Python mirror */
  FTT_ERR_OOM = 2,       /* -> MemoryError */
  FTT_ERR_NONFINITE = 3, /* -> ValueError("matrix entries must be finite") */
  FTT_ERR_CUDA = 4,      /* -> RuntimeError */
  FTT_ERR_NOCONV = 5     /* -> numpy.linalg.LinAlgError (SVD did not converge) */
} ftt_status;

typedef struct ftt_ctx ftt_ctx;

/* ------------------------------------------------------------ context */
const char *ftt_version(void);
const char *ftt_last_error(void);
/* stream: a cudaStream_t passed as an opaque pointer (0 = legacy default). */
int ftt_create(int device, void *stream, ftt_ctx **ctx_out);
int ftt_destroy(ftt_ctx *ctx);
int ftt_set_stream(ftt_ctx *ctx, void *stream);
/* Deferred status checks (on != 0): the narrow QR kernels OR their
 * non-finite-input flag into a device word instead of reading it back per
 * call; ftt_take_status reads and clears it (bit 0 = non-finite input).
 * Used by the decomposition driver, whose inputs are validated finite up
 * front (tensor.py:129-146), to drop one host round trip per QR-sweep step. */
int ftt_set_deferred_checks(ftt_ctx *ctx, int32_t on);
int ftt_take_status(ftt_ctx *ctx, int32_t *flags_out);
/* Host round trips (device->host reads that wait on the stream) since
 * creation and the host milliseconds spent blocked in them (instrumentation). */
int ftt_sync_stats(const ftt_ctx *ctx, int64_t *syncs_out, double *wait_ms_out);
/* Number of kernels this context launched since creation (instrumentation). */
int64_t ftt_kernel_launches(const ftt_ctx *ctx);
/* Live kernel timing for the roofline report: while enabled, every launch of
 * an instrumented kernel is bracketed by CUDA events on the context stream
 * and tagged with its class and algorithmic bytes / flops.  Enabling clears
 * the records.  Classes: 0 sort passes, 1 key build + histogram, 2 segment,
 * 3 deparallelisation sweep, 4 scatters, 5 DMMA GEMM, 6 QR panel,
 * 7 Jacobi step, 8 tt_entries. */
int ftt_profile_enable(ftt_ctx *ctx, int enable);
int ftt_profile_read(ftt_ctx *ctx, int32_t tag, double *ms_out,
                     int64_t *launches_out, double *bytes_out,
                     double *flops_out);
/* fp64 tensor-pipe (DMMA) peak microbenchmark: TFLOP/s over `iters`
 * back-to-back mma.sync.m8n8k4.f64 per warp on every SM. */
int ftt_bench_dmma(ftt_ctx *ctx, int64_t iters, double *tflops_out);

/* ---------------------------------------------------- input side (host) */
/* COO text reader (formats.py:47-100, ingest_coo): header "# shape n1 ...
 * nd", then d 1-based indices and a value per nonempty line.  Host memory
 * only (no context, no GPU).  The whole reference contract is decided here:
 * Python text-mode line splitting (\n, \r\n, \r), str.split() tokens,
 * Python int()/float() literal grammar, the reference's order of checks.
 * On success *coords_out (nnz x d, 0-based) and *vals_out are malloc'd --
 * release them with ftt_free_host.  A rejected file returns
 * FTT_ERR_INVALID and fills *err (err->text malloc'd, ftt_free_host); the
 * Python layer words the reference's FormatError from it. */
enum {
  FTT_COO_IO = 1,         /* unreadable file */
  FTT_COO_EMPTY = 2,      /* zero bytes: "empty file, missing shape header" */
  FTT_COO_HEADER = 3,     /* line 1 is not "# shape n1 ... nd" */
  FTT_COO_SHAPE = 4,      /* extents fail int()/check_shape; text = line 1 */
  FTT_COO_FIELDS = 5,     /* count = number of fields on the line */
  FTT_COO_UNPARSABLE = 6, /* text = the line */
  FTT_COO_RANGE = 7,      /* mode = 0-based mode, text = the index token */
  FTT_COO_NONFINITE = 8,  /* text = the value token */
  FTT_COO_NONASCII = 9    /* count = byte offset, mode = the byte */
};
typedef struct ftt_coo_error {
  int32_t kind;
  int32_t mode;
  int64_t line;  /* 1-based */
  int64_t count;
  char *text;
  int64_t text_len;
} ftt_coo_error;
int ftt_parse_coo_text(const char *path, int32_t max_d, int32_t *d_out,
                       int64_t *dims_out, int64_t *nnz_out,
                       int64_t **coords_out, double **vals_out,
                       ftt_coo_error *err);
/* MatrixMarket coordinate reader (formats.py:103-127).  *banner_out
 * classifies line 1 (FTT_MM_*); for `real general|symmetric` files the body
 * is read strictly (0-based rows/cols, symmetric entries expanded: stored
 * entries in file order, then mirrored off-diagonal ones in file order --
 * scipy.io.mmread's order) into malloc'd arrays.  FTT_ERR_INVALID = a body
 * the strict reader does not accept: the caller defers to scipy.io.mmread,
 * the library the reference reads with, for its result or error text. */
enum {
  FTT_MM_NOT_MM = 1,
  FTT_MM_OBJECT = 2,
  FTT_MM_FORMAT = 3,
  FTT_MM_FIELD = 4,
  FTT_MM_SYMMETRY = 5,
  FTT_MM_GENERAL = 6,
  FTT_MM_SYMMETRIC = 7
};
int ftt_parse_mm_text(const char *path, int32_t *banner_out, int64_t *shape_out,
                      int64_t *nnz_out, int64_t **rows_out, int64_t **cols_out,
                      double **vals_out);
void ftt_free_host(void *p);

/* ---------------------------------------------------- index path (int) */

/* The device COO as its canonical C-order linear index (SparseTensor's
 * sort key, tensor.py:75-100 linearize): one int64 per nonzero,
 * strictly increasing.  The entry points below read it instead of the
 * nnz x d coordinates (8 B per nonzero instead of 8d). */
int ftt_linearize(ftt_ctx *ctx, const int64_t *coords, int64_t nnz, int32_t d,
                  const int64_t *dims_host, int64_t *lin_out);
/* select_p's fiber counts for every pivot (fasttt.py:536-541) from lin:
 * pivots p >= ceil(d/2) on lin itself (chunks aligned to the prefix over
 * modes < ceil(d/2)), the others on lin bucketed by a hash of the suffix
 * over modes >= ceil(d/2) (two radix passes), shared-memory hash sets per
 * chunk.  coords (optional) serve pivots whose groups exceed a chunk. */
int ftt_fiber_counts_lin(ftt_ctx *ctx, const int64_t *lin, const int64_t *coords,
                         int64_t nnz, int32_t d, const int64_t *dims_host,
                         int64_t *counts_host);
/* ftt_extract_fibers (tensor.py:374-403) with the fiber keys built from
 * lin. */
int ftt_extract_fibers_lin(ftt_ctx *ctx, const int64_t *lin, const double *values,
                           int64_t nnz, int32_t d, const int64_t *dims_host,
                           int32_t pivot, int64_t *fixed_lin, int64_t *indptr,
                           int64_t *fiber_of, int64_t *pivot_index,
                           double *values_out, int64_t *num_fibers_out);

/* Distinct fixed tuples for one pivot mode: the fiber count R_p computed
 * by select_p, `np.unique(linearize(rest_dims, coords[:, rest])).size`
 * (fasttt.py:537-541).  coords: nnz x d int64 row-major. */
int ftt_fiber_count(ftt_ctx *ctx, const int64_t *coords, int64_t nnz,
                    int32_t d, const int64_t *dims_host, int32_t pivot,
                    int64_t *count_out);

/* Fiber counts for every pivot 0..d-1 (select_p's loop, fasttt.py:536-541),
 * written to counts_host[d]. */
int ftt_fiber_counts_all(ftt_ctx *ctx, const int64_t *coords, int64_t nnz,
                         int32_t d, const int64_t *dims_host,
                         int64_t *counts_host);

/* extract_nonzero_fibers (tensor.py:374-403) / build_structured_tt
 * (fasttt.py:170-178).  Sorts by key lin(fixed)*n_p + i_p (the lexsort of
 * tensor.py:387-389 as one integer key) and segments where the fixed tuple
 * changes.  Outputs (capacity nnz, resp. nnz+1):
 *   fixed_lin[R]   C-order linear index of the fixed tuple over rest dims
 *   indptr[R+1]    fiber f owns entries indptr[f]..indptr[f+1]
 *   fiber_of[nnz]  fiber id of every sorted entry (may be NULL)
 *   pivot_index[nnz], values_out[nnz]  entries in fiber order
 * num_fibers_out (host) receives R. */
/* delinearize (tensor.py:75-100): coords_out (nnz x d int64 row-major) =
 * the C-order digits of lin[i] over dims.  The drop-in moves a canonical
 * COO to the device as its linear index (8 B per nonzero) and rebuilds the
 * coordinate rows here. */
int ftt_delinearize(ftt_ctx *ctx, const int64_t *lin, int64_t nnz, int32_t d,
                    const int64_t *dims_host, int64_t *coords_out);
int ftt_extract_fibers(ftt_ctx *ctx, const int64_t *coords,
                       const double *values, int64_t nnz, int32_t d,
                       const int64_t *dims_host, int32_t pivot,
                       int64_t *fixed_lin, int64_t *indptr, int64_t *fiber_of,
                       int64_t *pivot_index, double *values_out,
                       int64_t *num_fibers_out);
/* tensorize_matrix (ttformat.py:414-433) on the device: matrix entries
 * (rows[e], cols[e], vals[e]) -> the fused d-way tensor with f_i = x_i *
 * col_dims[i] + y_i (x, y the row / column digits over row_dims / col_dims),
 * in canonical form: C-order sorted, duplicates summed in input order (the
 * reference's tocsr() coalescing), zero sums dropped (tensor.py:147-153).
 * coords_out (nnz x d int64 row-major) and vals_out hold nnz entries;
 * *nnz_out = entries kept.  FTT_ERR_INVALID for an entry outside the
 * factored extents. */
int ftt_tensorize_matrix(ftt_ctx *ctx, int64_t nnz, const int64_t *rows,
                         const int64_t *cols, const double *vals, int32_t d,
                         const int64_t *row_dims, const int64_t *col_dims,
                         int64_t *coords_out, double *vals_out, int64_t *nnz_out);

/* depar_quasi_perm (fasttt.py:148-167): kept = ascending distinct rows of
 * col_to_row, t_map[j] = rank of col_to_row[j] among kept.  kept capacity
 * min(n_rows, n_cols). n_kept_out (host). */
int ftt_depar_quasi_perm(ftt_ctx *ctx, int64_t n_rows, int64_t n_cols,
                         const int64_t *col_to_row, int64_t *kept,
                         int64_t *t_map, int64_t *n_kept_out);
/* depar_general (fasttt.py:96-145): floating-point deparallelisation of the
 * rows x cols column-major M (ld ldm).  Columns in order; column j is
 * parallel to kept basis column i when |u - c b_i|^2 <= tol^2 |u|^2 with
 * c = (b_i . u) / |b_i|^2, the lowest such i wins; zero columns are dropped
 * (t_row = -1).  Outputs: kept[0..width) = basis columns of M
 * (first-occurrence order), t_row / t_coeff per column (the single nonzero
 * of t's column j), width_at[j] = basis width when column j was visited
 * (the reference's float_ops accounting), *width_out.  Device arrays of
 * cols entries each. */
int ftt_depar_general(ftt_ctx *ctx, int64_t rows, int64_t cols, const double *M,
                      int64_t ldm, double tol, int64_t *kept, int64_t *t_row,
                      double *t_coeff, int64_t *width_at, int64_t *width_out);

/* One step of _index_sweeps (fasttt.py:192-210) fused with its key build:
 *   side 0 (left of pivot):  key[f] = map_in[f] * n_k + i_k(f)
 *   side 1 (right of pivot): key[f] = i_k(f) * r_other + map_in[f]
 * with i_k(f) = (fixed_lin[f] / stride_k) % n_k, and n_rows = r_other*n_k.
 * map_in may be NULL (all zeros, first step of a side).  Then
 * depar_quasi_perm on (n_rows, R, key): kept (capacity min(R, n_rows)),
 * map_out[R], n_kept_out (host). */
int ftt_index_sweep_step(ftt_ctx *ctx, int32_t side, const int64_t *fixed_lin,
                         int64_t R, int64_t stride_k, int64_t n_k,
                         const int64_t *map_in, int64_t r_other,
                         int64_t *kept, int64_t *map_out,
                         int64_t *n_kept_out);
/* Every deparallelisation step of _index_sweeps (fasttt.py:181-211) in one
 * call and one host round trip: steps s = left modes 0..p-1, then right modes
 * d-1..p+1; each step's kept count stays on the device and feeds the next
 * step's key.  kept[s] (device, min(R, bound_s) entries with bound_s =
 * min(R, product of the modes already swept on that side) * n_k) and maps[s]
 * (device, R entries) are the same arrays ftt_index_sweep_step produces;
 * n_kept_out[s] the kept counts.  FTT_ERR_INVALID when a bound exceeds the
 * flag path's limits (the caller then steps with ftt_index_sweep_step). */
int ftt_index_sweeps_all(ftt_ctx *ctx, const int64_t *fixed_lin, int64_t R,
                         int32_t d, const int64_t *dims, int32_t pivot,
                         int64_t *const *kept, int64_t *const *maps,
                         int64_t *n_kept_out);

/* Per-fiber coordinate of one rest mode: (fixed_lin / stride) % n
 * (StructuredTT.mode_index, ttformat.py:322-327). */
int ftt_mode_index(ftt_ctx *ctx, const int64_t *fixed_lin, int64_t R,
                   int64_t stride, int64_t n, int64_t *out);

/* Pivot core of parallel_vector_round (fasttt.py:256-259): zero-fills the
 * dense r_prev x n_p x r_next C-order core and scatters
 * core[t_map[f], pivot_index[e], s_map[f]] = values[e] for every entry e of
 * fiber f = fiber_of[e].  t_map / s_map may be NULL (all zeros).  Also
 * returns the 2-norm of the values (the _budget_norm of fasttt.py:359-361)
 * in norm_out (host) when norm_out != NULL. */
int ftt_pivot_core_scatter(ftt_ctx *ctx, int64_t nnz, const int64_t *fiber_of,
                           const int64_t *pivot_index, const double *values,
                           const int64_t *t_map, const int64_t *s_map,
                           int64_t r_prev, int64_t n_p, int64_t r_next,
                           double *core, double *norm_out);

/* Dense 0/1 side cores (fasttt.py:246-255), materialised only for the
 * standalone parallel_vector_round API and the capped error measure.
 * side 0: core (r_other, n, K) with core[kept[j]//n, kept[j]%n, j] = 1
 * side 1: core (K, n, r_other) with core[j, kept[j]//r_other, kept[j]%r_other] = 1 */
int ftt_side_core_dense(ftt_ctx *ctx, int32_t side, const int64_t *kept,
                        int64_t K, int64_t n, int64_t r_other, double *core);

/* --------------------------------------------- carries into 0/1 cores */
/* First-sweep carry into a right 0/1 core (fasttt.py:340-341 with the core
 * of :251-255): dst (rank x ncols_new, row-major) = 0, then
 * dst[a, kept[j]] = src[a*lds + j] for j < K. */
int ftt_scatter_cols(ftt_ctx *ctx, int64_t rank, int64_t K, const int64_t *kept,
                     const double *src, int64_t lds, int64_t ncols_new,
                     double *dst);
/* Second-sweep carry into a left 0/1 core (fasttt.py:354-355 with the core
 * of :246-250): dst (nrows_new x rank, row-major) = 0, then
 * dst[kept[j], :] = src[j*lds + 0..rank). */
int ftt_scatter_rows(ftt_ctx *ctx, int64_t K, int64_t rank, const int64_t *kept,
                     const double *src, int64_t lds, int64_t nrows_new,
                     double *dst);

/* ------------------------------------------------------ dense fp64 */
/* C = alpha*op(A)*op(B) + beta*C, column-major, BLAS dgemm semantics
 * (trans = 0 'N', 1 'T').  Replaces np.tensordot / np.einsum / @ on the
 * dense carries (fasttt.py:341, 347, 355). DMMA (mma.sync m8n8k4 f64). */
int ftt_dgemm(ftt_ctx *ctx, int32_t transa, int32_t transb, int64_t m,
              int64_t n, int64_t k, double alpha, const double *A, int64_t lda,
              const double *B, int64_t ldb, double beta, double *C,
              int64_t ldc);

/* max |G - I| over an n x n column-major Gram (the orthonormality test of
 * _check_pivot_orthogonal, fasttt.py:303-321), to out_host. */
int ftt_orth_defect(ftt_ctx *ctx, int64_t n, const double *G, int64_t ldg,
                    double *out_host);

/* dst (cols x rows, ldd) = src^T (src rows x cols, lds), column-major. */
int ftt_transpose(ftt_ctx *ctx, int64_t rows, int64_t cols, const double *src,
                  int64_t lds, double *dst, int64_t ldd);

/* qr_economic (linalg.py:128-140): reduced Householder QR of the m x n
 * column-major A; Q (m x k) and R (k x n), k = min(m, n), diag(R) >= 0.
 * A is not modified. Non-finite input -> FTT_ERR_NONFINITE. */
int ftt_qr_f64(ftt_ctx *ctx, int64_t m, int64_t n, const double *A,
               int64_t lda, double *Q, int64_t ldq, double *R, int64_t ldr);

/* _full_svd (linalg.py:48-53), phase 1: thin SVD of the m x n matrix A,
 * column-major (a_row_major = 0) or row-major / numpy C-order
 * (a_row_major = 1), leading dimension lda (Householder QR + one-sided block
 * Jacobi).  Writes the k = min(m,n) singular values, descending, to s_host.
 * Factors stay in the context for phase 2.  A is not modified. */
int ftt_svd_f64(ftt_ctx *ctx, int64_t m, int64_t n, const double *A,
                int64_t lda, int32_t a_row_major, double *s_host);
/* Certified low-rank phase 1 (an accelerator for svd_truncate_delta on
 * numerically low-rank operands): A_tall ~= Q B with Q an orthonormal basis
 * of the numerically spanning columns of the sketch A_tall Omega (Omega a
 * deterministic k-column test matrix, k <= min(m,n) / 2), B = Q^T A_tall,
 * and the residual R = A_tall - Q B evaluated explicitly:
 * rest2_host = ||R||_F^2.  The singular values of B go to s_host (at most k;
 * the rest stay untouched) and phase 2 (ftt_svd_vectors) returns Q U_B /
 * V_B.  Every true tail sum of A_tall lies in [tail_B, tail_B + rest2]
 * (A^T A = B^T B + R^T R).  *accepted = 2 when rest2 <=
 * min(max(1e-8 delta2, nA eps^2 ||A||_F^2), 1e-6 delta2) -- below the
 * rounding noise of a full backward-stable SVD's tails (the reference's
 * gesdd); = 1 when only rest2 <= 1e-6 delta2 (the caller may use it when
 * the tail rule of linalg.py:97-99 decides the same rank at both ends of
 * the interval); = 0 otherwise, and the caller runs ftt_svd_f64.
 * delta2 = delta^2 of the truncation step. */
int ftt_svd_lowrank_f64(ftt_ctx *ctx, int64_t m, int64_t n, const double *A,
                        int64_t lda, int32_t a_row_major, int64_t k,
                        double delta2, double *s_host, double *rest2_host,
                        int32_t *accepted);
/* The same certified low-rank phase 1 on the pivot core of
 * parallel_vector_round (fasttt.py:256-259) given by its entries instead of
 * the dense core: the operand is M = core.reshape(r_prev * n_p, r_next)
 * (m = r_prev * n_p, n = r_next), entry e at row t_map[f] * n_p +
 * pivot_index[e], column s_map[f] (f = fiber_of[e]; t_map / s_map NULL for
 * r_prev / r_next = 1), value values[e] -- the FiberSet arrays of
 * ftt_extract_fibers and the maps of ftt_index_sweep_step.  Y, B and the
 * residual energy (over every element of M, zeros included) are computed
 * from the entries; k <= 64.  Phase 2 is ftt_svd_vectors as above.  A
 * rejected certificate (accepted = 0) leaves the caller to densify the core
 * (ftt_pivot_core_scatter) for ftt_svd_f64. */
int ftt_svd_lowrank_sparse_f64(ftt_ctx *ctx, int64_t m, int64_t n, int64_t nnz,
                               const int64_t *fiber_of,
                               const int64_t *pivot_index,
                               const double *values, const int64_t *t_map,
                               const int64_t *s_map, int64_t n_p, int64_t k,
                               double delta2, double *s_host,
                               double *rest2_host, int32_t *accepted);
/* Phase 2: the leading `rank` singular triplets of the last ftt_svd_f64, with
 * the sign convention of _fix_signs (linalg.py:56-63) applied to U: U (m x
 * rank) and V (n x rank, i.e. vt.T), each column- or row-major per its flag;
 * scale_v != 0 multiplies column j of V by s[j] (the carry vt.T * s of
 * fasttt.py:340/354).  U or V may be NULL. */
int ftt_svd_vectors(ftt_ctx *ctx, int64_t rank, double *U, int64_t ldu,
                    int32_t u_row_major, double *V, int64_t ldv,
                    int32_t v_row_major, int32_t scale_v);

/* sum of squares of x (n values), written to out_host (frobenius_norm,
 * tensor.py:298-302, and the sparse_inner_error dot, fasttt.py:596-599 when
 * y != NULL: sum x*y). */
int ftt_dot(ftt_ctx *ctx, int64_t n, const double *x, const double *y,
            double *out_host);

/* tt_entries (ttformat.py:124-136): out[i] = G0[:, c[i,0], :] @ ... @
 * G_{d-1}[:, c[i,d-1], :] for n coordinates (n x d int64 row-major).
 * cores_host[k] is a device pointer to the C-order (r_k, n_k, r_{k+1}) core;
 * ranks_host has d+1 entries, dims_host d. */
int ftt_tt_entries(ftt_ctx *ctx, int32_t d, const int64_t *dims_host,
                   const int64_t *ranks_host, const double *const *cores_host,
                   const int64_t *coords, int64_t n, double *out);
/* Frobenius norm of the same train description (tt_norm, ttformat.py:198-203):
 * the train contracted with itself core by core (two DMMA GEMMs per core). */
int ftt_tt_norm(ftt_ctx *ctx, int32_t d, const int64_t *dims_host,
                const int64_t *ranks_host, const double *const *cores_host,
                double *norm_out);
/* sparse_inner_error's data terms (fasttt.py:587-602) in one round trip:
 * out_host[0] = <values, entries> over n points, out_host[1] = ||t||^2 of the
 * train (dims / ranks / cores as ftt_tt_entries). */
int ftt_inner_terms(ftt_ctx *ctx, int64_t n, const double *values,
                    const double *entries, int32_t d, const int64_t *dims_host,
                    const int64_t *ranks_host, const double *const *cores_host,
                    double *out_host);
/* <a, b> of the report's inner-product identity (fasttt.py:587-602) on the
 * index structure fasttt holds: the sweep's kept rows (left steps 0..p-1,
 * then right steps d-1..p+1, in that order, kept_counts alike) name the
 * distinct prefixes / suffixes, t_map / s_map each fiber's; b's prefix and
 * suffix vectors are built once per distinct prefix / suffix and each
 * nonzero costs one length-r_p dot.  indptr (R + 1) / pivot_index /
 * values: the fibers and their nonzeros in fiber order
 * (ftt_extract_fibers); cores: the rounded train b (ranks[0] = ranks[d] =
 * 1).  *out_host = sum_e values[e] b(e). */
int ftt_inner_structured(ftt_ctx *ctx, int32_t d, const int64_t *dims,
                         const int64_t *ranks, const double *const *cores,
                         int32_t pivot, const int64_t *const *kept,
                         const int64_t *kept_counts, int64_t R,
                         const int64_t *indptr, const int64_t *pivot_index,
                         const double *values, const int64_t *t_map,
                         const int64_t *s_map, double *out_host);

/* ------------------------------------------------------ rounding driver */
/* One core of the structured train handed to ftt_sweep_rounding:
 *  kind 0: dense (r0, n, r1) C-order buffer `data` (caller-owned, read only);
 *  kind 1 / 2: left / right 0/1 core as its kept rows (`kept`, K entries,
 *    r_other = the bond on the far side), the SideCore of the Python mirror;
 *  kind 3: the pivot core given by its entries (ftt_sparse_pivot). */
typedef struct {
  int32_t kind;
  int64_t r0, n, r1;
  double *data;
  const int64_t *kept;
  int64_t K, r_other;
} ftt_core_desc;
/* The pivot core's entries (fasttt.py:256-259): value[e] at
 * (t_map[fiber_of[e]], pivot_index[e], s_map[fiber_of[e]]); NULL maps for
 * unit edge bonds. */
typedef struct {
  int64_t nnz;
  const int64_t *fiber_of, *pivot_index;
  const double *values;
  const int64_t *t_map, *s_map;
  /* optional (0 / NULL when unknown): the fiber structure the entries came
   * from (tensor.py:374-403: num_fibers fibers, fiber f holds entries
   * indptr[f] .. indptr[f+1]) -- lets the first step index its operand by
   * fiber instead of sorting the entries */
  int64_t num_fibers;
  const int64_t *indptr;
} ftt_sparse_pivot;
/* _sweep_rounding (fasttt.py:324-356) in one call: SVD sweep p..d-2, QR
 * sweep d-1..p+1, SVD sweep p..1, with policy 0 = static (delta per step,
 * fasttt.py:364-386), 1 = dynamic (left / right budgets re-absorbed,
 * fasttt.py:389-428), 2 = fixed ranks (targets[d+1], fasttt.py:431-453);
 * interval_ok lets a static step accept a low-rank certificate whose
 * interval decides the same rank (dense.dev_svd_truncate).  Output cores:
 * out_ptrs[k] fresh device buffers (release with ftt_free_device), shapes
 * out_shapes[3k..3k+2]; *zero_out = 1 (and no outputs) when a truncation
 * reaches rank 0 (the zero train, fasttt.py:337-338, 351-352). */
int ftt_sweep_rounding(ftt_ctx *ctx, int32_t d, int32_t pivot,
                       const ftt_core_desc *cores, const ftt_sparse_pivot *sp,
                       int32_t policy, double delta, double left, double right,
                       const int64_t *targets, int32_t interval_ok,
                       double **out_ptrs, int64_t *out_shapes, int32_t *zero_out);
/* Release a device buffer returned by ftt_sweep_rounding (stream-ordered). */
int ftt_free_device(ftt_ctx *ctx, void *p);

/* How many truncation steps of this process ran the certified low-rank
 * path on a scattered carry's compact form and were accepted (the operand
 * of fasttt.py:334-341 after a 0/1 core, never materialised; test probe). */
int64_t ftt_scatter_steps(void);

/* The canonical linear index of the NEXT call that reads `lin`
 * (ftt_fiber_counts_lin, ftt_extract_fibers_lin, ftt_fasttt_lin) is still
 * arriving from the host: chunk j, lin[0 .. ends[j]), is present once the
 * cudaEvent_t events[j] has fired (ends ascending, <= 8 chunks).  select_p's
 * forward counts (fasttt.py:536-541) then start on the chunks present and
 * overlap the rest of the transfer; every other reader waits for the last
 * event.  The chunk list is consumed by that call. */
int ftt_set_lin_chunks(ftt_ctx *ctx, int32_t nchunks, const int64_t *ends, void *const *events);

/* ------------------------------------------------------- fasttt driver */
/* What ftt_fasttt_lin hands back.  Device buffers the caller releases with
 * ftt_free_device: fiber_slab (fixed_lin, indptr, fiber_of, pivot_index,
 * values_f point into it), kept_slab (step s's kept rows at kept_off[s],
 * step_counts[s] entries; steps ordered as ftt_index_sweeps_all: modes
 * 0..p-1 then d-1..p+1), maps_slab (step s's fiber map at s * max(R, 1)),
 * and the output train: out_slab when non-NULL (every core inside it, back
 * to back in mode order), else each out_cores[k] on its own. */
typedef struct {
  int32_t pivot;        /* the pivot used (select_p's choice when asked) */
  int32_t zero;         /* a truncation reached rank 0: the cores are zeros (1, n_k, 1) */
  int32_t fallback;     /* 1: nothing was produced, use the step-by-step entry points */
  int32_t inner_valid;  /* dot / nb hold the report's terms */
  int32_t lazy_pivot;   /* the pivot core stayed as its entries */
  int32_t status_flags; /* ftt_take_status (bit 0: non-finite input) */
  int64_t num_fibers;
  int64_t step_counts[32];
  int64_t kept_off[32];
  int64_t pivot_shape[3];
  int64_t out_shapes[96];
  int64_t out_total;    /* elements of the output train */
  double na2, pnorm, dot, nb;
  void *fiber_slab;
  int64_t *fixed_lin, *indptr, *fiber_of, *pivot_index;
  double *values_f;
  int64_t *kept_slab, *maps_slab;
  double *out_slab;
  double *out_cores[32];
} ftt_fasttt_result;
/* fasttt (fasttt.py:634-749) for static (mode 0) and dynamic (mode 1)
 * budgets in one call on the canonical COO (lin strictly increasing +
 * values, device): select_p when pivot < 0 (fasttt.py:501-558, exact-int
 * cost model), extract_nonzero_fibers, _index_sweeps, the structured train
 * with the pivot core kept as its entries below 2 % density, the rounding
 * sweeps, and with report != 0 the inner-product identity's terms
 * (na2 = |a|^2, dot = <a, b>, nb = |b|).  values_ready (optional
 * cudaEvent_t) is waited for after select_p, before the values are read.
 * Sets res->fallback instead of failing when an extent or bound exceeds
 * the fused path's limits. */
int ftt_fasttt_lin(ftt_ctx *ctx, const int64_t *lin, const double *values,
                   int64_t nnz, int32_t d, const int64_t *dims, int32_t pivot,
                   int32_t mode, double eps, double c_svd, int32_t report,
                   void *values_ready, ftt_fasttt_result *res);

#ifdef __cplusplus
}
#endif
#endif /* FASTTT_B200_H */
