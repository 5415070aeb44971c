// Blocked Householder QR in fp64 (qr_economic, linalg.py:128-140, and the
// QR factor under every SVD of the rounding sweeps).
//
// Two-level blocking:
//  * inner panels of QR_NBI = 32 columns are factored column by column by ONE
//    cooperative kernel spread over up to 148 CTAs: each CTA owns a row chunk,
//    one pass computes the partial norm of the column and its dots with the
//    remaining panel columns, a grid barrier reduces them (fixed order, so
//    the result is deterministic and identical in every CTA), a second pass
//    applies the reflector.  LAPACK dlarfg conventions (beta = -sign(alpha)
//    * norm, tau = (beta - alpha) / beta, tau = 0 when the tail is zero).
//  * outer blocks of QR_NBO = 128 columns update the trailing matrix with the
//    compact-WY form  C <- C - V T^T (V^T C)  as three DMMA GEMMs; the T
//    factors are kept so that Q can be applied later (qr_apply_q).
#include <cooperative_groups.h>

#include <algorithm>

#include "ftt_dense.cuh"
#include "ftt_small.cuh"

namespace cg = cooperative_groups;

namespace ftt {
namespace {

constexpr int PT = 256;
constexpr int PW = PT / 32;
constexpr int PSLOTS = 34;  // alpha-row (32) + xx + spare

// 32 per-lane accumulators -> lane l receives the warp-wide sum of slot l,
// in 31 shuffles (halving exchange: at offset s each lane keeps the upper or
// lower s slots by bit s of its lane id and adds the partner's copy).
__device__ __forceinline__ double warp_reduce_scatter32(double (&acc)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int j = 0; j < s; ++j) {
      const double send = upper ? acc[j] : acc[j + s];
      const double keep = upper ? acc[j + s] : acc[j];
      acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return acc[0];
}

// Factor the mp x jb panel (jb <= 32) at A (lda).  partials: gridDim.x * PSLOTS.
__global__ void __launch_bounds__(PT) k_panel(int64_t mp, int jb, double *__restrict__ A,
                                              int64_t lda, double *__restrict__ tau,
                                              double *__restrict__ partials) {
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const int64_t chunk = (mp + G - 1) / G;
  const int64_t r0 = (int64_t)blockIdx.x * chunk;
  const int64_t r1 = min(mp, r0 + chunk);
  __shared__ double s_red[PW][33];
  __shared__ double s_dot[33];
  __shared__ double s_row[33];  // row c of the panel, read before any update
  __shared__ double s_w[33];
  __shared__ double s_sc[3];

  for (int c = 0; c < jb; ++c) {
    const int nj = jb - c;  // columns c..jb-1 (slot 0 = the column itself)
    if (tid < nj) s_row[tid] = A[c + (int64_t)(c + tid) * lda];
    double acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0;
    const double *colc = A + (int64_t)c * lda;
    for (int64_t i = max(r0, (int64_t)c + 1) + tid; i < r1; i += PT) {
      double x = colc[i];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nj) acc[j] += x * colc[i + (int64_t)j * lda];
    }
    s_red[warp][lane] = warp_reduce_scatter32(acc, lane);  // lane j <- warp total of slot j
    __syncthreads();
    if (tid < nj) {
      double t = 0.0;
      for (int w = 0; w < PW; ++w) t += s_red[w][tid];
      partials[(int64_t)blockIdx.x * PSLOTS + tid] = t;
    }
    grid.sync();
    if (tid < nj) {
      double t = 0.0;
      for (int g = 0; g < G; ++g) t += partials[(int64_t)g * PSLOTS + tid];
      s_dot[tid] = t;
    }
    __syncthreads();
    if (tid == 0) {
      double alpha = s_row[0], xx = s_dot[0];
      double tc, beta, scal;
      if (xx == 0.0) {
        tc = 0.0;
        beta = alpha;
        scal = 0.0;
      } else {
        beta = -copysign(sqrt(alpha * alpha + xx), alpha);
        tc = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      s_sc[0] = tc;
      s_sc[1] = beta;
      s_sc[2] = scal;
      if (blockIdx.x == 0) tau[c] = tc;
    }
    __syncthreads();
    const double tc = s_sc[0], beta = s_sc[1], scal = s_sc[2];
    if (tid >= 1 && tid < nj) s_w[tid] = tc * (s_row[tid] + scal * s_dot[tid]);
    __syncthreads();
    if (tc != 0.0) {
      double *colw = A + (int64_t)c * lda;
      for (int64_t i = max(r0, (int64_t)c + 1) + tid; i < r1; i += PT) {
        double v = colw[i] * scal;
        colw[i] = v;
        for (int j = 1; j < nj; ++j) colw[i + (int64_t)j * lda] -= s_w[j] * v;
      }
    }
    if (c >= r0 && c < r1) {  // the diagonal row lives in this CTA
      if (tid == 0) A[c + (int64_t)c * lda] = beta;
      if (tc != 0.0 && tid >= 1 && tid < nj) A[c + (int64_t)(c + tid) * lda] -= s_w[tid];
    }
    grid.sync();
  }
}

// V (mp x jb, ld ldv) = unit lower trapezoid of the factored panel.
__global__ void k_extract_v(int64_t mp, int jb, const double *__restrict__ A, int64_t lda,
                            double *__restrict__ V, int64_t ldv) {
  int64_t total = mp * jb;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / mp, i = t - j * mp;
    double v = i > j ? A[i + j * lda] : (i == j ? 1.0 : 0.0);
    V[i + j * ldv] = v;
  }
}


// Blocked dlarft for nb <= 128 in one CTA of 1024 threads, T staged in
// shared memory: 32x32 diagonal blocks by the scalar recurrence (one warp
// each, in parallel), then block columns j = 1.. with
// T[0:j, j] = -T[0:j, 0:j] (VtV[0:j, j] T_jj)   (T12 = -T11 V1^T V2 T22).
// Replaces the 128-step sequential recurrence (~90 us per call) by ~4
// dependent phases.
constexpr int LF_MAX = 128;
__global__ void __launch_bounds__(1024) k_larft_blocked(int nb, const double *__restrict__ VtV,
                                                        int64_t ldg, const double *__restrict__ tau,
                                                        double *__restrict__ Tout, int64_t ldt) {
  extern __shared__ double lf[];
  double *T = lf;                  // nb x nb, column-major, ld = nb
  double *W = lf + LF_MAX * LF_MAX;  // <= 96 x 32, column-major, ld = 96
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < nb * nb; e += blockDim.x) T[e] = 0.0;
  __syncthreads();
  const int nblk = (nb + 31) / 32;
  if (warp < nblk) {
    const int b0 = warp * 32, bs = min(32, nb - b0);
    for (int i = 0; i < bs; ++i) {
      const double ti = tau[b0 + i];
      if (lane < i) {
        double v = 0.0;
        if (ti != 0.0) {
          for (int l = lane; l < i; ++l)
            v += T[(b0 + lane) + (b0 + l) * nb] * VtV[(b0 + l) + (int64_t)(b0 + i) * ldg];
          v = -ti * v;
        }
        T[(b0 + lane) + (b0 + i) * nb] = v;
      }
      if (lane == i) T[(b0 + i) + (b0 + i) * nb] = ti;
      __syncwarp();
    }
  }
  __syncthreads();
  for (int j = 1; j < nblk; ++j) {
    const int c0 = j * 32, cs = min(32, nb - c0);
    // W = VtV[0:c0, c0:c0+cs] * T_jj (T_jj upper triangular)
    for (int e = tid; e < c0 * cs; e += blockDim.x) {
      const int r = e % c0, c = e / c0;
      double v = 0.0;
      for (int k = 0; k <= c; ++k) v += VtV[r + (int64_t)(c0 + k) * ldg] * T[(c0 + k) + (c0 + c) * nb];
      W[r + c * 96] = v;
    }
    __syncthreads();
    // T[0:c0, c0:c0+cs] = -T[0:c0, 0:c0] * W (upper triangular T)
    for (int e = tid; e < c0 * cs; e += blockDim.x) {
      const int r = e % c0, c = e / c0;
      double v = 0.0;
      for (int l = r; l < c0; ++l) v += T[r + l * nb] * W[l + c * 96];
      T[r + (c0 + c) * nb] = -v;
    }
    __syncthreads();
  }
  for (int e = tid; e < nb * nb; e += blockDim.x) Tout[(e % nb) + (int64_t)(e / nb) * ldt] = T[e];
}

__global__ void k_finite(int64_t m, int64_t n, const double *__restrict__ A, int64_t lda, int *bad) {
  int64_t total = m * n;
  int b = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / m, i = t - j * m;
    if (!isfinite(A[i + j * lda])) b = 1;
  }
  if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

__global__ void k_copy_matrix(int64_t m, int64_t n, const double *__restrict__ src, int64_t lds,
                              double *__restrict__ dst, int64_t ldd) {
  int64_t total = m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / m, i = t - j * m;
    dst[i + j * ldd] = src[i + j * lds];
  }
}

// R (k x n, ldr) from the factored A; diag sign flips d_i = sign(R_ii) (0->1)
// are applied to the rows of R here and to the columns of Q by k_scale_q.
__global__ void k_extract_r(int64_t k, int64_t n, const double *__restrict__ A, int64_t lda,
                            double *__restrict__ R, int64_t ldr) {
  int64_t total = k * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / k, i = t - j * k;
    double v = 0.0;
    if (j >= i) {
      double d = A[i + i * lda];
      double sg = d < 0.0 ? -1.0 : 1.0;
      v = sg * A[i + j * lda];
    }
    R[i + j * ldr] = v;
  }
}

__global__ void k_identity(int64_t m, int64_t k, double *Z, int64_t ldz) {
  int64_t total = m * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / m, i = t - j * m;
    Z[i + j * ldz] = i == j ? 1.0 : 0.0;
  }
}

__global__ void k_scale_q(int64_t m, int64_t k, const double *__restrict__ A, int64_t lda,
                          double *__restrict__ Q, int64_t ldq) {
  int64_t total = m * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / m, i = t - j * m;
    if (A[j + j * lda] < 0.0) Q[i + j * ldq] = -Q[i + j * ldq];
  }
}

// ---------------------------------------------------------------------------
// Shared-memory-resident panel: the mp x jb panel is split by rows over the
// CTAs of ONE thread-block cluster (MODE 0, reductions over DSMEM, one
// cluster barrier per column) or over a cooperative grid of <= 148 CTAs
// (MODE 1, partials through global memory, one grid barrier per column).
// Every column step then reads shared memory only; the panel is loaded and
// stored once.  Partials are double-buffered so one barrier per column is
// enough (a CTA can only overwrite buffer b after every CTA passed the next
// barrier, i.e. finished reading b).
constexpr int RES_ROWS = 768;  // rows per CTA: 768 x 32 x 8 B = 192 KiB

template <int MODE>
__global__ void __launch_bounds__(PT) k_panel_res(int64_t mp, int jb, double *__restrict__ A,
                                                  int64_t lda, double *__restrict__ tau,
                                                  double *__restrict__ gpart) {
  extern __shared__ double sm[];
  __shared__ double s_red[PW][33];
  __shared__ double s_part[2][PSLOTS];
  __shared__ double s_rowc[2][PSLOTS];
  __shared__ double s_dot[33], s_row[33], s_w[33], s_sc[3];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = gridDim.x, me = blockIdx.x;
  const int64_t chunk = (mp + nb - 1) / nb;
  const int64_t r0 = (int64_t)me * chunk;
  const int64_t r1 = min(mp, r0 + chunk);
  const int nr = (int)max((int64_t)0, r1 - r0);
  const int64_t ld = chunk;
#pragma unroll 8
  for (int j = 0; j < jb; ++j) {  // unrolled over columns: many loads in flight
    const double *src = A + r0 + (int64_t)j * lda;
    double *dst = sm + (int64_t)j * ld;
    for (int li = tid; li < nr; li += PT) dst[li] = src[li];
  }
  __syncthreads();
  for (int c = 0; c < jb; ++c) {
    const int buf = c & 1, nj = jb - c;
    double acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0;
    const int lo = (int)(max(r0, (int64_t)c + 1) - r0);
    const double *colc = sm + (int64_t)c * ld;
    for (int li = lo + tid; li < nr; li += PT) {
      double x = colc[li];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nj) acc[j] += x * colc[li + (int64_t)j * ld];
    }
    s_red[warp][lane] = warp_reduce_scatter32(acc, lane);  // lane j <- warp total of slot j
    __syncthreads();
    const bool owner = c >= r0 && c < r1;
    if (tid < nj) {
      double t = 0.0;
      for (int w = 0; w < PW; ++w) t += s_red[w][tid];
      double rv = owner ? sm[(c - r0) + (int64_t)(c + tid) * ld] : 0.0;
      if (MODE == 0) {
        s_part[buf][tid] = t;
        if (owner) s_rowc[buf][tid] = rv;
      } else {
        gpart[((int64_t)buf * nb + me) * PSLOTS + tid] = t;
        if (owner) gpart[((int64_t)2 * nb) * PSLOTS + buf * PSLOTS + tid] = rv;
      }
    }
    if (MODE == 0) {
      cg::this_cluster().sync();
    } else {
      cg::this_grid().sync();
    }
    const int own = (int)(c / chunk);
    {
      // warp w sums the partials of CTAs q = w, w+8, ... (slot = lane); the 8
      // warp sums are then added in warp order -- fixed order, so every CTA
      // computes bit-identical scalars
      double t = 0.0;
      if (lane < nj) {
#pragma unroll 4
        for (int q = warp; q < nb; q += PW) {
          if (MODE == 0) {
            const double *rp = cg::this_cluster().map_shared_rank(&s_part[buf][0], q);
            t += rp[lane];
          } else {
            t += gpart[((int64_t)buf * nb + q) * PSLOTS + lane];
          }
        }
      }
      s_red[warp][lane] = t;
    }
    __syncthreads();
    if (tid < nj) {
      double t = 0.0;
      for (int w = 0; w < PW; ++w) t += s_red[w][tid];
      s_dot[tid] = t;
      if (MODE == 0) {
        s_row[tid] = cg::this_cluster().map_shared_rank(&s_rowc[buf][0], own)[tid];
      } else {
        s_row[tid] = gpart[((int64_t)2 * nb) * PSLOTS + buf * PSLOTS + tid];
      }
    }
    __syncthreads();
    if (tid == 0) {
      double alpha = s_row[0], xx = s_dot[0];
      double tc, beta, scal;
      if (xx == 0.0) {
        tc = 0.0;
        beta = alpha;
        scal = 0.0;
      } else {
        beta = -copysign(sqrt(alpha * alpha + xx), alpha);
        tc = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      s_sc[0] = tc;
      s_sc[1] = beta;
      s_sc[2] = scal;
      if (me == 0) tau[c] = tc;
    }
    __syncthreads();
    const double tc = s_sc[0], beta = s_sc[1], scal = s_sc[2];
    if (tid >= 1 && tid < nj) s_w[tid] = tc * (s_row[tid] + scal * s_dot[tid]);
    __syncthreads();
    if (tc != 0.0) {
      double *colw = sm + (int64_t)c * ld;
      for (int li = lo + tid; li < nr; li += PT) {
        double v = colw[li] * scal;
        colw[li] = v;
        for (int j = 1; j < nj; ++j) colw[li + (int64_t)j * ld] -= s_w[j] * v;
      }
    }
    if (owner) {
      if (tid == 0) sm[(c - r0) + (int64_t)c * ld] = beta;
      if (tc != 0.0 && tid >= 1 && tid < nj) sm[(c - r0) + (int64_t)(c + tid) * ld] -= s_w[tid];
    }
    __syncthreads();
  }
#pragma unroll 8
  for (int j = 0; j < jb; ++j) {
    double *dst = A + r0 + (int64_t)j * lda;
    const double *src = sm + (int64_t)j * ld;
    for (int li = tid; li < nr; li += PT) dst[li] = src[li];
  }
  if (MODE == 0) cg::this_cluster().sync();  // keep our smem alive for DSMEM readers
}

int panel_grid(ftt_ctx *ctx, int64_t mp) {
  static int max_blocks = 0;
  if (!max_blocks) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_panel, PT, 0);
    if (per_sm < 1) per_sm = 1;
    max_blocks = per_sm * ctx->num_sms;
  }
  int64_t g = ceil_div(mp, 2048);
  g = std::max<int64_t>(1, std::min<int64_t>(g, std::min(max_blocks, ctx->num_sms)));
  return (int)g;
}

int launch_panel(ftt_ctx *ctx, int64_t mp, int jb, double *A, int64_t lda, double *tau,
                 double *partials) {
  static bool attrs = false;
  if (!attrs) {
    FTT_CUDA(cudaFuncSetAttribute(k_panel_res<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  RES_ROWS * QR_NBI * 8));
    FTT_CUDA(cudaFuncSetAttribute(k_panel_res<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  RES_ROWS * QR_NBI * 8));
    FTT_CUDA(cudaFuncSetAttribute(k_panel_res<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attrs = true;
  }
  const int64_t nblocks = ceil_div(mp, RES_ROWS);
  if (nblocks <= 16) {
    // one cluster; DSMEM reductions
    const int C = (int)std::max<int64_t>(nblocks, 1);
    const size_t smem = (size_t)ceil_div(mp, C) * jb * 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(PT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FTT_CUDA(cudaLaunchKernelEx(&cfg, k_panel_res<0>, mp, jb, A, lda, tau, partials));
    FTT_LAUNCHED(ctx);
    return FTT_OK;
  }
  if (nblocks <= ctx->num_sms) {
    // cooperative grid, one CTA per SM (192 KiB smem each)
    int G = (int)nblocks;
    size_t smem = (size_t)ceil_div(mp, G) * jb * 8;
    void *args[] = {&mp, &jb, &A, &lda, &tau, &partials};
    FTT_CUDA(cudaLaunchCooperativeKernel((const void *)k_panel_res<1>, dim3(G), dim3(PT), args, smem,
                                         ctx->stream));
    FTT_LAUNCHED(ctx);
    return FTT_OK;
  }
  int g = panel_grid(ctx, mp);
  void *args[] = {&mp, &jb, &A, &lda, &tau, &partials};
  FTT_CUDA(cudaLaunchCooperativeKernel((const void *)k_panel, dim3(g), dim3(PT), args, 0,
                                       ctx->stream));
  FTT_LAUNCHED(ctx);
  return FTT_OK;
}

struct QrWs {
  double *V, *VtV, *T, *W, *W2, *part, *splitk;
  size_t splitk_elems;
};

constexpr size_t SPLITK_ELEMS = (size_t)2 * 296 * 64 * 64 + 4096;

bool carve(double *ws, size_t ws_elems, int64_t m, int64_t n, QrWs *q) {
  size_t off = 0;
  auto grab = [&](size_t e) {
    double *p = ws + off;
    off += (e + 31) / 32 * 32;
    return p;
  };
  q->V = grab((size_t)std::max<int64_t>(m, 1) * QR_NBO);
  q->VtV = grab((size_t)QR_NBO * QR_NBO);
  q->T = grab((size_t)QR_NBO * QR_NBO);
  q->W = grab((size_t)QR_NBO * std::max<int64_t>(n, 1));
  q->W2 = grab((size_t)QR_NBO * std::max<int64_t>(n, 1));
  q->part = grab((size_t)kNumSMs * 8 * PSLOTS);
  q->splitk = grab(SPLITK_ELEMS);
  q->splitk_elems = SPLITK_ELEMS;
  return off <= ws_elems;
}

// C (mp x nc) <- (I - V T' V^T) C with T' = T^T (trans=1) or T (trans=0).
int apply_block(ftt_ctx *ctx, int64_t mp, int64_t nc, int jb, const double *V, int64_t ldv,
                const double *T, int64_t ldt, int trans, double *C, int64_t ldc, QrWs &w) {
  if (nc <= 0 || mp <= 0) return FTT_OK;
  FTT_CHECK(gemm(ctx, 1, 0, jb, nc, mp, 1.0, V, ldv, C, ldc, 0.0, w.W, jb, w.splitk, w.splitk_elems));
  FTT_CHECK(gemm(ctx, trans, 0, jb, nc, jb, 1.0, T, ldt, w.W, jb, 0.0, w.W2, jb, w.splitk,
                 w.splitk_elems));
  FTT_CHECK(gemm(ctx, 0, 0, mp, nc, jb, -1.0, V, ldv, w.W2, jb, 1.0, C, ldc, w.splitk,
                 w.splitk_elems));
  return FTT_OK;
}

int build_t(ftt_ctx *ctx, int64_t mp, int jb, const double *A, int64_t lda, const double *tau,
            double *T, int64_t ldt, QrWs &w) {
  k_extract_v<<<grid_for(mp * jb, 256, 4), 256, 0, ctx->stream>>>(mp, jb, A, lda, w.V, mp);
  FTT_LAUNCHED(ctx);
  FTT_CHECK(gemm(ctx, 1, 0, jb, jb, mp, 1.0, w.V, mp, w.V, mp, 0.0, w.VtV, jb, w.splitk,
                 w.splitk_elems));
  static bool attr = false;
  const size_t smem = sizeof(double) * (LF_MAX * LF_MAX + 96 * 32);
  if (!attr) {
    FTT_CUDA(cudaFuncSetAttribute(k_larft_blocked, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr = true;
  }
  k_larft_blocked<<<1, 1024, smem, ctx->stream>>>(jb, w.VtV, jb, tau, T, ldt);
  FTT_LAUNCHED(ctx);
  return FTT_OK;
}

}  // namespace

size_t qr_workspace_elems(int64_t m, int64_t n) {
  return (size_t)std::max<int64_t>(m, 1) * QR_NBO + 2 * QR_NBO * QR_NBO +
         2 * (size_t)QR_NBO * std::max<int64_t>(n, 1) + kNumSMs * 8 * PSLOTS + SPLITK_ELEMS + 256;
}

size_t qr_tblk_elems(int64_t m, int64_t n) {
  int64_t k = std::min(m, n);
  return (size_t)std::max<int64_t>(ceil_div(k, QR_NBO), 1) * QR_NBO * QR_NBO;
}

size_t qr_apply_workspace_elems(int64_t m, int64_t n, int64_t r) {
  return qr_workspace_elems(m, std::max(n, r));
}

int qr_factor(ftt_ctx *ctx, int64_t m, int64_t n, double *A, int64_t lda, double *tau, double *Tblk,
              double *ws, size_t ws_elems) {
  QrWs w;
  if (!carve(ws, ws_elems, m, n, &w)) {
    set_error("qr_factor: workspace too small");
    return FTT_ERR_INVALID;
  }
  const int64_t k = std::min(m, n);
  for (int64_t J = 0; J < k; J += QR_NBO) {
    const int jbo = (int)std::min<int64_t>(QR_NBO, k - J);
    for (int64_t j = J; j < J + jbo; j += QR_NBI) {
      const int jb = (int)std::min<int64_t>(QR_NBI, J + jbo - j);
      double *Aj = A + j + j * lda;
      {
        const int pb = prof_begin(ctx);
        FTT_CHECK(launch_panel(ctx, m - j, jb, Aj, lda, tau + j, w.part));
        // Householder panel: ~2 (m-j) jb^2 flops; reads+writes the panel once
        prof_end(ctx, pb, PT_QR_PANEL, 16.0 * (double)(m - j) * jb,
                 2.0 * (double)(m - j) * jb * jb);
      }
      const int64_t nrest = (J + jbo) - (j + jb);
      if (nrest > 0) {
        FTT_CHECK(build_t(ctx, m - j, jb, Aj, lda, tau + j, w.T, jb, w));
        FTT_CHECK(apply_block(ctx, m - j, nrest, jb, w.V, m - j, w.T, jb, 1, Aj + jb * lda, lda, w));
      }
    }
    double *TJ = Tblk + (J / QR_NBO) * QR_NBO * QR_NBO;
    double *AJ = A + J + J * lda;
    FTT_CHECK(build_t(ctx, m - J, jbo, AJ, lda, tau + J, TJ, jbo, w));
    if (J + jbo < n)
      FTT_CHECK(apply_block(ctx, m - J, n - (J + jbo), jbo, w.V, m - J, TJ, jbo, 1, AJ + jbo * lda,
                            lda, w));
  }
  return FTT_OK;
}

int qr_build_tblk(ftt_ctx *ctx, int64_t m, int64_t n, const double *A, int64_t lda,
                  const double *tau, double *Tblk, double *ws, size_t ws_elems) {
  QrWs w;
  if (!carve(ws, ws_elems, m, n, &w)) {
    set_error("qr_build_tblk: workspace too small");
    return FTT_ERR_INVALID;
  }
  const int64_t k = std::min(m, n);
  for (int64_t J = 0; J < k; J += QR_NBO) {
    const int jbo = (int)std::min<int64_t>(QR_NBO, k - J);
    FTT_CHECK(build_t(ctx, m - J, jbo, A + J + J * lda, lda, tau + J,
                      Tblk + (J / QR_NBO) * QR_NBO * QR_NBO, jbo, w));
  }
  return FTT_OK;
}

int qr_apply_q(ftt_ctx *ctx, int64_t m, int64_t n, const double *A, int64_t lda, const double *Tblk,
               int64_t r, double *Z, int64_t ldz, double *ws, size_t ws_elems) {
  QrWs w;
  if (!carve(ws, ws_elems, m, std::max(n, r), &w)) {
    set_error("qr_apply_q: workspace too small");
    return FTT_ERR_INVALID;
  }
  const int64_t k = std::min(m, n);
  if (k == 0 || r == 0) return FTT_OK;
  int64_t last = ((k - 1) / QR_NBO) * QR_NBO;
  for (int64_t J = last; J >= 0; J -= QR_NBO) {
    const int jbo = (int)std::min<int64_t>(QR_NBO, k - J);
    const double *TJ = Tblk + (J / QR_NBO) * QR_NBO * QR_NBO;
    k_extract_v<<<grid_for((m - J) * jbo, 256, 4), 256, 0, ctx->stream>>>(m - J, jbo, A + J + J * lda,
                                                                         lda, w.V, m - J);
    FTT_LAUNCHED(ctx);
    FTT_CHECK(apply_block(ctx, m - J, r, jbo, w.V, m - J, TJ, jbo, 0, Z + J, ldz, w));
  }
  return FTT_OK;
}

int check_finite(ftt_ctx *ctx, int64_t m, int64_t n, const double *A, int64_t lda, bool *ok) {
  *ok = true;
  if (m * n == 0) return FTT_OK;
  int *bad = static_cast<int *>(arena_take(ctx, 256));
  if (!bad) {
    set_error("check_finite: arena too small");
    return FTT_ERR_INVALID;
  }
  FTT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
  k_finite<<<grid_for(m * n, 256, 4), 256, 0, ctx->stream>>>(m, n, A, lda, bad);
  FTT_LAUNCHED(ctx);
  int h = 0;
  FTT_CHECK(copy_to_host(ctx, &h, bad, sizeof(int)));
  *ok = h == 0;
  return FTT_OK;
}

int copy_matrix(ftt_ctx *ctx, int64_t m, int64_t n, const double *src, int64_t lds, double *dst,
                int64_t ldd) {
  if (m * n == 0) return FTT_OK;
  if (lds == m && ldd == m) {
    FTT_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, ctx->stream));
    return FTT_OK;
  }
  k_copy_matrix<<<grid_for(m * n, 256, 4), 256, 0, ctx->stream>>>(m, n, src, lds, dst, ldd);
  FTT_LAUNCHED(ctx);
  return FTT_OK;
}

int launch_identity(ftt_ctx *ctx, int64_t m, int64_t k, double *Z, int64_t ldz) {
  if (m * k == 0) return FTT_OK;
  k_identity<<<grid_for(m * k, 256, 4), 256, 0, ctx->stream>>>(m, k, Z, ldz);
  FTT_LAUNCHED(ctx);
  return FTT_OK;
}

}  // namespace ftt

using namespace ftt;

extern "C" int ftt_qr_f64(ftt_ctx *ctx, int64_t m, int64_t n, const double *A, int64_t lda,
                          double *Q, int64_t ldq, double *R, int64_t ldr) {
  if (!ctx || m < 0 || n < 0) return FTT_ERR_INVALID;
  const int64_t k = std::min(m, n);
  if (k == 0) return FTT_OK;
  static const bool no_small = getenv("FTT_NO_SMALL") != nullptr;
  if (!no_small && tsqr_ok(m, n)) {
    // narrow: TSQR tree of CTA-local Householder QRs (ftt_small.cu)
    double *Qt = Q;
    if (!Qt) FTT_CHECK(owned_alloc(ctx, (void **)&Qt, 8 * (size_t)m * n));
    const int rc = tsqr_q(ctx, m, n, A, lda, 0, Qt, Q ? ldq : m, R, ldr);
    if (!Q) owned_free(ctx, Qt);
    return rc;
  }
  size_t wse = qr_workspace_elems(m, std::max(n, k));
  size_t need = align_up(8 * (size_t)m * n) + align_up(8 * (size_t)k) +
                align_up(8 * qr_tblk_elems(m, n)) + align_up(8 * wse) + 1024;
  FTT_CHECK(arena_reserve(ctx, need));
  bool ok = true;
  FTT_CHECK(check_finite(ctx, m, n, A, lda, &ok));
  if (!ok) {
    set_error("matrix entries must be finite");
    return FTT_ERR_NONFINITE;
  }
  double *Af = take<double>(ctx, (size_t)m * n);
  double *tau = take<double>(ctx, k);
  double *Tb = take<double>(ctx, qr_tblk_elems(m, n));
  double *ws = take<double>(ctx, wse);
  if (!Af || !tau || !Tb || !ws) {
    set_error("ftt_qr_f64: arena too small");
    return FTT_ERR_INVALID;
  }
  FTT_CHECK(copy_matrix(ctx, m, n, A, lda, Af, m));
  FTT_CHECK(qr_factor(ctx, m, n, Af, m, tau, Tb, ws, wse));
  if (R) {
    k_extract_r<<<grid_for(k * n, 256, 4), 256, 0, ctx->stream>>>(k, n, Af, m, R, ldr);
    FTT_LAUNCHED(ctx);
  }
  if (Q) {
    FTT_CHECK(launch_identity(ctx, m, k, Q, ldq));
    FTT_CHECK(qr_apply_q(ctx, m, n, Af, m, Tb, k, Q, ldq, ws, wse));
    k_scale_q<<<grid_for(m * k, 256, 4), 256, 0, ctx->stream>>>(m, k, Af, m, Q, ldq);
    FTT_LAUNCHED(ctx);
  }
  return FTT_OK;
}
