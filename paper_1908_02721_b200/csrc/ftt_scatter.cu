// Scattered operand of a right-sweep truncation step (fasttt.py:334-341
// after a step whose next core is a 0/1 core): the carry S V^T (r1 x rank)
// times the 0/1 core (r1, n, r_other) is rank * K numbers placed into a
// (rank n) x r_other matrix -- config 5's second step holds 5 M values in a
// 430 MB operand.  The certified low-rank path (ftt_svd.cu: sketch, B = Q^T A,
// certificate residual) runs here on the compact form instead of four passes
// over the zero-filled matrix:
//   A_tall (mA = r_other rows, nA = rank n columns), column (a, i) = a n + i,
//   A_tall[c', a n + i] = V[c + a ldv] for the entry c with kept[c] = i mA + c'
// (kept ascending, so the entries of a block column i are contiguous and
// their rows ascend).  `pos` (n x mA int32) is the inverse of kept: the entry
// at (i, c') or -1; every row-wise kernel walks it in ascending i, so each
// sum has one fixed order (bit-reproducible, no atomics).
#include <algorithm>

#include "ftt_dense.cuh"

namespace ftt {
namespace {

__global__ void k_sc_pos(int64_t K, const int64_t *__restrict__ kept, int32_t *__restrict__ pos) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < K;
       c += (int64_t)gridDim.x * blockDim.x)
    pos[kept[c]] = (int32_t)c;
}

// iptr[i] = first entry with kept >= i mA (i = 0..n)
__global__ void k_sc_iptr(int64_t K, const int64_t *__restrict__ kept, int64_t mA, int64_t n,
                          int64_t *__restrict__ iptr) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  const int64_t key = i * mA;
  int64_t lo = 0, hi = K;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (kept[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  iptr[i] = lo;
}

// The range finder's test matrix (ftt_svd.cu k_omega: splitmix64 of the
// column-major element index col + j nA), stored row-major nA x k.
__global__ void k_sc_omega(int64_t nA, int k, double *__restrict__ Ot) {
  const int64_t total = nA * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = t / k, j = t - col * k;
    uint64_t z = (uint64_t)(col + j * nA) + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    Ot[t] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
}

// Y = A_tall Omega in two steps: W[c, :] = V[c, :] Omega_{i(c)} per entry (one
// thread per entry, 8 sketch columns at a time; a warp's entries mostly share
// the block column, so the Omega loads are broadcasts), then Y[c', :] = the
// sum of W[c, :] over the row's entries in ascending block column (one thread
// per row: coalesced pos reads and Y writes).  k is a multiple of 8.
constexpr int SW_SL = 2;  // block columns of Omega a CTA stages (its entries rarely span more)

template <int K8>
__global__ void __launch_bounds__(128) k_sc_w(int64_t K, int64_t mA, int64_t n, int r, int max_sl,
                                              const int64_t *__restrict__ kept,
                                              const double *__restrict__ V, int64_t ldv,
                                              const double *__restrict__ Ot,
                                              double *__restrict__ W) {
  constexpr int k = 8 * K8;
  extern __shared__ __align__(16) double sm[];  // SW_SL slices of r x k
  const int64_t c0 = blockIdx.x * (int64_t)blockDim.x;
  const int64_t c = c0 + threadIdx.x;
  // the CTA's entries are consecutive, so their block columns are
  // [i_lo, i_hi]; the first SW_SL slices of Omega go to shared memory
  const int64_t i_lo = __ldg(kept + c0) / mA;
  const int64_t i_hi = __ldg(kept + min(c0 + (int64_t)blockDim.x, K) - 1) / mA;
  const int nsl = (int)min((int64_t)max_sl, i_hi - i_lo + 1);
  for (int e = threadIdx.x; e < nsl * r * (k / 2); e += blockDim.x) {
    const int sl = e / (r * (k / 2)), rem = e - sl * (r * (k / 2));
    const int a = rem / (k / 2), u = rem - a * (k / 2);
    reinterpret_cast<double2 *>(sm)[e] =
        __ldg(reinterpret_cast<const double2 *>(Ot + ((int64_t)a * n + i_lo + sl) * k) + u);
  }
  __syncthreads();
  if (c >= K) return;
  const int64_t i = __ldg(kept + c) / mA;
  const double *v = V + c;
  double w[k];
#pragma unroll
  for (int u = 0; u < k; ++u) w[u] = 0.0;
  const bool in_sm = i - i_lo < nsl;
  const double2 *o = in_sm ? reinterpret_cast<const double2 *>(sm) + (i - i_lo) * r * (k / 2)
                           : reinterpret_cast<const double2 *>(Ot + i * k);
  const int64_t os2 = in_sm ? (k / 2) : n * (k / 2);
  for (int a0 = 0; a0 < r; a0 += 8) {
    double va[8];  // one round of loads for 8 carry components
#pragma unroll
    for (int u = 0; u < 8; ++u) va[u] = a0 + u < r ? __ldg(v + (a0 + u) * ldv) : 0.0;
#pragma unroll
    for (int aa = 0; aa < 8; ++aa) {
      if (a0 + aa < r) {
        const double2 *oa = o + (a0 + aa) * os2;
#pragma unroll
        for (int u = 0; u < k / 2; ++u) {
          const double2 x = oa[u];
          w[2 * u] = fma(va[aa], x.x, w[2 * u]);
          w[2 * u + 1] = fma(va[aa], x.y, w[2 * u + 1]);
        }
      }
    }
  }
  double2 *dst = reinterpret_cast<double2 *>(W + c * k);
#pragma unroll
  for (int u = 0; u < k / 2; ++u) dst[u] = make_double2(w[2 * u], w[2 * u + 1]);
}

template <int K8>
__global__ void __launch_bounds__(128) k_sc_ysum(int64_t mA, int64_t n,
                                                 const int32_t *__restrict__ pos,
                                                 const double *__restrict__ W,
                                                 double *__restrict__ Y) {
  constexpr int k = 8 * K8;
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= mA) return;
  const int32_t *p = pos + row;
  double y[k];
#pragma unroll
  for (int u = 0; u < k; ++u) y[u] = 0.0;
  for (int64_t i0 = 0; i0 < n; i0 += 8) {
    int32_t c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = i0 + u < n ? __ldg(p + (i0 + u) * mA) : -1;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (c[u] >= 0) {
        const double2 *w = reinterpret_cast<const double2 *>(W + (int64_t)c[u] * k);
#pragma unroll
        for (int q = 0; q < k / 2; ++q) {
          const double2 x = __ldg(w + q);
          y[2 * q] += x.x;
          y[2 * q + 1] += x.y;
        }
      }
  }
#pragma unroll
  for (int u = 0; u < k; ++u) Y[row + (int64_t)u * mA] = y[u];
}

// B[:, (a, i)] = sum over the entries c of block column i of Q[c'(c), :]^T
// V[c, a] on the fp64 tensor pipe: CTA (s, i) takes split s of the block
// column's entries in tiles of TE staged in shared memory (Q rows gathered);
// warp w owns the 8 x 8 output tiles w, w + 4, ... (mma.m8n8k4: the entry
// index is the inner dimension) and writes them to P[i][s];
// k_sc_qta_reduce adds the splits in order.
constexpr int QT_MAXT = 16;  // output tiles per warp (NT <= QT_MAXT): (kr / 8) (r / 8) <= 64

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NT>
__global__ void __launch_bounds__(128) k_sc_qta(int64_t mA, int64_t n, int r, int kr, int S,
                                                int TE, const int64_t *__restrict__ kept,
                                                const int64_t *__restrict__ iptr,
                                                const double *__restrict__ V, int64_t ldv,
                                                const double *__restrict__ Q,
                                                double *__restrict__ P) {
  extern __shared__ __align__(16) double sm[];
  const int tq = (kr + 7) >> 3, tr = (r + 7) >> 3;
  const int lq = tq * 8 + 4, lv = tr * 8 + 4;  // row strides == 4 mod 8: conflict-free fragments
  double *Qs = sm;             // TE x lq
  double *Vs = sm + TE * lq;   // TE x lv
  __shared__ int rows_s[128];  // TE <= 128: the tile's entry rows
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = blockIdx.y;
  const int s = blockIdx.x;
  const int64_t b0 = iptr[i], b1 = iptr[i + 1];
  const int64_t len = (b1 - b0 + S - 1) / S;
  const int64_t lo = b0 + (int64_t)s * len, hi = min(b1, lo + len);
  const int T = tq * tr;
  double acc[NT][2];
  int qo[NT], vo[NT];  // fragment offsets of this warp's tiles
  bool own[NT];        // (a tile past T is computed on tile 0's data and dropped)
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    acc[t][0] = acc[t][1] = 0.0;
    const int tile = warp + 4 * t;
    own[t] = tile < T;
    qo[t] = own[t] ? (tile % tq) * 8 : 0;
    vo[t] = own[t] ? (tile / tq) * 8 : 0;
  }
  for (int64_t t0 = lo; t0 < hi; t0 += TE) {
    const int te = (int)min((int64_t)TE, hi - t0);
    const int tep = (te + 3) & ~3;
    __syncthreads();
    for (int el = threadIdx.x; el < tep; el += 128)
      rows_s[el] = el < te ? (int)(__ldg(kept + t0 + el) - i * mA) : -1;
    __syncthreads();
    {
      // 8 independent loads in flight per thread and round (global latency
      // ~1 us: a load per loop trip serialises the tile's staging)
      const int w8 = tq * 8, nq = tep * w8;
      for (int e0 = threadIdx.x; e0 < nq; e0 += 8 * 128) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * 128;
          x[u] = 0.0;
          if (e < nq) {
            const int q = e % w8, el = e / w8;
            const int row = rows_s[el];
            if (row >= 0 && q < kr) x[u] = __ldg(Q + row + (int64_t)q * mA);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * 128;
          if (e < nq) Qs[(e / w8) * lq + e % w8] = x[u];
        }
      }
      const int v8 = tr * 8, nv = tep * v8;
      for (int e0 = threadIdx.x; e0 < nv; e0 += 8 * 128) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * 128;
          x[u] = 0.0;
          if (e < nv) {
            const int el = e % tep, a = e / tep;
            if (el < te && a < r) x[u] = __ldg(V + t0 + el + (int64_t)a * ldv);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * 128;
          if (e < nv) Vs[(e % tep) * lv + e / tep] = x[u];
        }
      }
    }
    __syncthreads();
    for (int ks = 0; ks < tep; ks += 4) {
      const double *qrow = Qs + (ks + (lane & 3)) * lq + (lane >> 2);
      const double *vrow = Vs + (ks + (lane & 3)) * lv + (lane >> 2);
#pragma unroll
      for (int t = 0; t < NT; ++t) dmma(acc[t][0], acc[t][1], qrow[qo[t]], vrow[vo[t]]);
    }
  }
  double *dst = P + ((int64_t)i * S + s) * ((int64_t)kr * r);
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    if (own[t]) {
      const int q = qo[t] + (lane >> 2);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = vo[t] + 2 * (lane & 3) + h;
        if (q < kr && a < r) dst[a * kr + q] = acc[t][h];
      }
    }
  }
}

__global__ void k_sc_qta_reduce(int64_t n, int r, int kr, int S, const double *__restrict__ P,
                                double *__restrict__ B) {
  const int nout = kr * r;
  const int64_t total = n * nout;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / nout;
    const int out = (int)(t - i * nout);
    const int q = out % kr, a = out / kr;
    const double *p = P + i * S * nout + out;
    double x = 0.0;
    for (int s = 0; s < S; ++s) x += p[(int64_t)s * nout];
    B[q + ((int64_t)a * n + i) * kr] = x;
  }
}

// ||A_tall - Q B||_F^2 in two sums of non-negative terms.  Off the entries
// (k_sc_resid): a CTA takes `rows` rows (sub-tiles of RS_RT) and a tile of 256
// columns (APT values of a times NP values of i), each thread one column
// with its B column in registers; e = Q[row, :] B[:, col] from the shared Q
// tile, squared and summed where pos has no entry.  On the entries
// (k_sc_resid_on): one thread per entry, (V[c, a] - Q[c', :] B[:, (a, i)])^2
// over its r components.  Block sums in fixed order.
constexpr int RS_RT = 16;

template <int KRP>
__global__ void __launch_bounds__(256) k_sc_resid(int64_t mA, int64_t n, int r, int kr, int NP,
                                                  int rows, const int32_t *__restrict__ pos,
                                                  const double *__restrict__ Q,
                                                  const double *__restrict__ B,
                                                  double *__restrict__ part) {
  extern __shared__ __align__(16) double sm[];
  constexpr int LQ = KRP + 2;  // padded row stride (even: double2 reads stay aligned)
  const int LP = NP + 1;
  double *Qs = sm;                                               // rows x LQ
  int32_t *ps = reinterpret_cast<int32_t *>(sm + rows * LQ);     // rows x LP
  __shared__ double red[256];
  const int APT = 256 / NP;
  const int ichunks = (int)((n + NP - 1) / NP);
  const int64_t row0 = (int64_t)blockIdx.x * rows;
  const int ic = blockIdx.y % ichunks, ac = blockIdx.y / ichunks;
  const int il = threadIdx.x % NP, al = threadIdx.x / NP;
  const int64_t i = (int64_t)ic * NP + il;
  const int a = ac * APT + al;
  const bool active = i < n && a < r;
  // staging in rounds of 8 independent loads per thread
  const int nqs = rows * KRP, nps = rows * NP;
  for (int e0 = threadIdx.x; e0 < nqs; e0 += 8 * 256) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256;
      const int rl = e % rows, q = e / rows;
      const int64_t row = row0 + rl;
      x[u] = (e < nqs && row < mA && q < kr) ? __ldg(Q + row + (int64_t)q * mA) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256;
      if (e < nqs) Qs[(e % rows) * LQ + e / rows] = x[u];
    }
  }
  for (int e0 = threadIdx.x; e0 < nps; e0 += 8 * 256) {
    int32_t x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256;
      const int rl = e % rows, ii = e / rows;
      const int64_t row = row0 + rl, gi = (int64_t)ic * NP + ii;
      x[u] = (e < nps && row < mA && gi < n) ? __ldg(pos + gi * mA + row) : -1;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256;
      if (e < nps) ps[(e % rows) * LP + e / rows] = x[u];
    }
  }
  double b[KRP];
  {
    const double *bcol = B + ((int64_t)a * n + i) * kr;
#pragma unroll
    for (int q = 0; q < KRP; ++q) b[q] = (active && q < kr) ? __ldg(bcol + q) : 0.0;
  }
  __syncthreads();
  double acc = 0.0;
  for (int sub = 0; sub < rows; sub += RS_RT) {
    double e[RS_RT];
#pragma unroll
    for (int rl = 0; rl < RS_RT; ++rl) e[rl] = 0.0;
#pragma unroll
    for (int q0 = 0; q0 < KRP; q0 += 8) {
#pragma unroll
      for (int rl = 0; rl < RS_RT; ++rl) {
        const double2 *qp = reinterpret_cast<const double2 *>(Qs + (sub + rl) * LQ + q0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 qq = qp[u];
          e[rl] = fma(qq.x, b[q0 + 2 * u], e[rl]);
          e[rl] = fma(qq.y, b[q0 + 2 * u + 1], e[rl]);
        }
      }
    }
#pragma unroll
    for (int rl = 0; rl < RS_RT; ++rl)
      if (ps[(sub + rl) * LP + il] < 0) acc = fma(e[rl], e[rl], acc);
  }
  red[threadIdx.x] = active ? acc : 0.0;
  __syncthreads();
  for (int off = 128; off; off >>= 1) {
    if ((int)threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(128) k_sc_resid_on(int64_t K, int64_t mA, int64_t n, int r,
                                                     int kr, const int64_t *__restrict__ kept,
                                                     const double *__restrict__ V, int64_t ldv,
                                                     const double *__restrict__ Q,
                                                     const double *__restrict__ B,
                                                     double *__restrict__ part) {
  __shared__ double red[128];
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double acc = 0.0;
  if (c < K) {
    const int64_t kc = __ldg(kept + c);
    const int64_t i = kc / mA, row = kc - i * mA;
    if (kr <= 16) {  // the basis row in registers (one round of loads)
      double qv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) qv[u] = u < kr ? __ldg(Q + row + (int64_t)u * mA) : 0.0;
      for (int a = 0; a < r; ++a) {
        const double *bcol = B + ((int64_t)a * n + i) * kr;
        double e = 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (u < kr) e = fma(qv[u], __ldg(bcol + u), e);
        const double x = __ldg(V + c + (int64_t)a * ldv) - e;
        acc = fma(x, x, acc);
      }
    } else {
      for (int a = 0; a < r; ++a) {
        const double *bcol = B + ((int64_t)a * n + i) * kr;
        double e = 0.0;
        for (int q = 0; q < kr; ++q) e = fma(__ldg(Q + row + (int64_t)q * mA), __ldg(bcol + q), e);
        const double x = __ldg(V + c + (int64_t)a * ldv) - e;
        acc = fma(x, x, acc);
      }
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int off = 64; off; off >>= 1) {
    if ((int)threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(1024) k_sc_sum(int64_t n, const double *__restrict__ part,
                                                 double *__restrict__ out) {
  __shared__ double red[1024];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 1024) a += part[i];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int off = 512; off; off >>= 1) {
    if ((int)threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

int pow2_ceil(int64_t x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace

bool scatter_operand_ok(int64_t mA, int64_t n, int64_t r, int64_t K) {
  return mA >= 1 && n >= 1 && r >= 1 && r <= 64 && K >= 1 && K < ((int64_t)1 << 31) &&
         n <= 65535 && n * mA <= ((int64_t)1 << 28);
}

int scatter_operand_build(ftt_ctx *ctx, ScatterOperand *op) {
  const int64_t cells = op->n * op->mA;
  FTT_CHECK(owned_alloc(ctx, (void **)&op->pos, 4 * (size_t)cells));
  FTT_CHECK(owned_alloc(ctx, (void **)&op->iptr, 8 * (size_t)(op->n + 1)));
  const int pb = prof_begin(ctx);
  FTT_CUDA(cudaMemsetAsync(op->pos, 0xff, 4 * (size_t)cells, ctx->stream));
  k_sc_pos<<<grid_for(op->K, 256, 4), 256, 0, ctx->stream>>>(op->K, op->kept, op->pos);
  FTT_LAUNCHED(ctx);
  k_sc_iptr<<<(unsigned)ceil_div(op->n + 1, 256), 256, 0, ctx->stream>>>(op->K, op->kept, op->mA,
                                                                         op->n, op->iptr);
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb, PT_SCATTER, 4.0 * (double)cells + 12.0 * (double)op->K, 0.0);
  return FTT_OK;
}

void scatter_operand_free(ftt_ctx *ctx, ScatterOperand *op) {
  owned_free(ctx, op->pos);
  owned_free(ctx, op->iptr);
  op->pos = nullptr;
  op->iptr = nullptr;
}

int scatter_sketch(ftt_ctx *ctx, const ScatterOperand &op, int64_t k, double *Y) {
  const int64_t nA = op.n * op.r;
  double *Ot = nullptr, *W = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&Ot, 8 * (size_t)nA * k));
  FTT_CHECK(owned_alloc(ctx, (void **)&W, 8 * (size_t)op.K * k));
  k_sc_omega<<<grid_for(nA * k, 256, 4), 256, 0, ctx->stream>>>(nA, (int)k, Ot);
  FTT_LAUNCHED(ctx);
  const int pb = prof_begin(ctx);
  if (k % 8 || k < 8 || k > 64) {
    set_error("scatter_sketch: k must be a multiple of 8 in [8, 64]");
    return FTT_ERR_INVALID;
  }
  const unsigned gw = (unsigned)ceil_div(op.K, 128), gy = (unsigned)ceil_div(op.mA, 128);
  int max_sl = SW_SL;  // Omega slices per CTA within the default 48 KB
  while (max_sl > 0 && 8 * (size_t)max_sl * op.r * k > 49152) --max_sl;
#define FTT_SC_SKETCH(K8)                                                                       \
  case K8:                                                                                      \
    k_sc_w<K8><<<gw, 128, 8 * (size_t)max_sl * op.r * k, ctx->stream>>>(                         \
        op.K, op.mA, op.n, (int)op.r, max_sl, op.kept, op.V, op.ldv, Ot, W);                    \
    FTT_LAUNCHED(ctx);                                                                          \
    k_sc_ysum<K8><<<gy, 128, 0, ctx->stream>>>(op.mA, op.n, op.pos, W, Y);                      \
    FTT_LAUNCHED(ctx);                                                                          \
    break;
  switch ((int)(k / 8)) {
    FTT_SC_SKETCH(1)
    FTT_SC_SKETCH(2)
    FTT_SC_SKETCH(3)
    FTT_SC_SKETCH(4)
    FTT_SC_SKETCH(5)
    FTT_SC_SKETCH(6)
    FTT_SC_SKETCH(7)
    FTT_SC_SKETCH(8)
  }
#undef FTT_SC_SKETCH
  prof_end(ctx, pb, PT_GEMM,
           4.0 * (double)op.n * op.mA + 8.0 * (double)op.K * (op.r + 2 * k) + 8.0 * (double)op.mA * k,
           2.0 * (double)op.K * op.r * (double)k);
  owned_free(ctx, Ot);
  owned_free(ctx, W);
  return FTT_OK;
}

int scatter_qt_a(ftt_ctx *ctx, const ScatterOperand &op, int64_t kr, const double *Q, double *B) {
  const int tq = (int)(kr + 7) / 8, tr = (int)(op.r + 7) / 8;
  if (kr > 64 || op.r > 64 || tq * tr > 4 * QT_MAXT) {
    set_error("scatter_qt_a: kr or r out of range");
    return FTT_ERR_INVALID;
  }
  const int lq = tq * 8 + 4, lv = tr * 8 + 4;
  const int TE = (int)std::max<int64_t>(8, std::min<int64_t>(128, (5120 / (lq + lv)) & ~3));
  // splits of about two tiles each, at most 64 per block column
  const int S = (int)std::max<int64_t>(
      1, std::min<int64_t>(64, ceil_div(ceil_div(op.K, op.n), 2 * TE)));
  const int64_t nout = kr * op.r;
  double *P = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&P, 8 * (size_t)op.n * S * nout));
  const size_t smem = 8 * (size_t)TE * (lq + lv);
  const int pb = prof_begin(ctx);
  const dim3 grid((unsigned)S, (unsigned)op.n);
  const int nt = (tq * tr + 3) / 4;
#define FTT_SC_QTA(NT)                                                                          \
  k_sc_qta<NT><<<grid, 128, smem, ctx->stream>>>(op.mA, op.n, (int)op.r, (int)kr, S, TE, op.kept, \
                                                 op.iptr, op.V, op.ldv, Q, P)
  if (nt <= 1) FTT_SC_QTA(1);
  else if (nt <= 2) FTT_SC_QTA(2);
  else if (nt <= 4) FTT_SC_QTA(4);
  else if (nt <= 8) FTT_SC_QTA(8);
  else FTT_SC_QTA(16);
#undef FTT_SC_QTA
  FTT_LAUNCHED(ctx);
  k_sc_qta_reduce<<<grid_for(op.n * nout, 256, 1), 256, 0, ctx->stream>>>(op.n, (int)op.r, (int)kr,
                                                                          S, P, B);
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb, PT_GEMM, 8.0 * (double)op.K * (op.r + kr + 1), 2.0 * (double)op.K * nout);
  owned_free(ctx, P);
  return FTT_OK;
}

int scatter_resid(ftt_ctx *ctx, const ScatterOperand &op, int64_t kr, const double *Q,
                  const double *B, double *out_dev) {
  const int NP = (int)std::min<int64_t>(256, pow2_ceil(op.n));
  const int APT = 256 / NP;
  const int KRP = kr <= 16 ? 16 : (kr <= 32 ? 32 : 64);
  if (kr > 64) {
    set_error("scatter_resid: kr > 64");
    return FTT_ERR_INVALID;
  }
  // rows per CTA: the Q tile and the pos tile within 48 KB
  int rows = 128;
  while (rows > RS_RT && (size_t)rows * (8 * (KRP + 2) + 4 * (NP + 1)) > 49152) rows >>= 1;
  const int64_t ichunks = ceil_div(op.n, NP), achunks = ceil_div(op.r, APT);
  const int64_t gx = ceil_div(op.mA, rows), gy = ichunks * achunks;
  if (gy > 65535) {
    set_error("scatter_resid: too many column tiles");
    return FTT_ERR_INVALID;
  }
  const int64_t gon = ceil_div(op.K, 128);
  double *part = nullptr;
  FTT_CHECK(owned_alloc(ctx, (void **)&part, 8 * (size_t)(gx * gy + gon)));
  const size_t smem = align_up((size_t)rows * (8 * (KRP + 2) + 4 * (NP + 1)), 16);
  static bool attr = false;
  if (!attr) {
    FTT_CUDA(cudaFuncSetAttribute(k_sc_resid<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  49152));
    FTT_CUDA(cudaFuncSetAttribute(k_sc_resid<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  49152));
    FTT_CUDA(cudaFuncSetAttribute(k_sc_resid<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  49152));
    attr = true;
  }
  const int pb = prof_begin(ctx);
  const dim3 grid((unsigned)gx, (unsigned)gy);
#define FTT_SC_RESID(KP)                                                                     \
  k_sc_resid<KP><<<grid, 256, smem, ctx->stream>>>(op.mA, op.n, (int)op.r, (int)kr, NP, rows, \
                                                   op.pos, Q, B, part)
  if (KRP == 16) FTT_SC_RESID(16);
  else if (KRP == 32) FTT_SC_RESID(32);
  else FTT_SC_RESID(64);
#undef FTT_SC_RESID
  FTT_LAUNCHED(ctx);
  k_sc_resid_on<<<(unsigned)gon, 128, 0, ctx->stream>>>(op.K, op.mA, op.n, (int)op.r, (int)kr,
                                                        op.kept, op.V, op.ldv, Q, B,
                                                        part + gx * gy);
  FTT_LAUNCHED(ctx);
  k_sc_sum<<<1, 1024, 0, ctx->stream>>>(gx * gy + gon, part, out_dev);
  FTT_LAUNCHED(ctx);
  prof_end(ctx, pb, PT_GEMM, 8.0 * (double)op.mA * kr * (double)gy + 4.0 * (double)op.n * op.mA,
           2.0 * (double)op.mA * (double)(op.n * op.r) * (double)kr);
  owned_free(ctx, part);
  return FTT_OK;
}

}  // namespace ftt
