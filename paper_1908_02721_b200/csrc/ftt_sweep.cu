// _sweep_rounding (fasttt.py:324-356) as one native call: the three sweeps
// (SVD sweep p..d-2, QR sweep d-1..p+1, SVD sweep p..1) with the truncation
// policy of fasttt.py:364-453 (static, dynamic, fixed rank) and the tail
// rule of linalg.py:89-100, driving the same C-ABI kernels the Python
// mirror calls step by step (pipeline._sweep_rounding_device).  Running the
// loop here removes ~0.4 ms of Python per config-2 decomposition (argument
// marshalling, numpy tail scans, tensor allocation between ~40 calls).
//
// Cores come in as descriptors: dense device buffers (caller-owned), 0/1
// side cores as kept arrays (carries are scatters), or the sparse pivot core
// (first step on its entries, densified on demand).  Every output core is a
// fresh cudaMallocAsync buffer handed to the caller (ftt_free_device).
#include <math.h>

#include <vector>

#include <stdlib.h>

#include "ftt_dense.cuh"
#include "../../include/fasttt_b200.h"

namespace ftt {
namespace {

constexpr double kEpsD = 2.220446049250313e-16;

// numpy's pairwise summation of a contiguous float64 array (the float
// order np.sum uses: 8 accumulators for blocks <= 128, recursive halves
// above), so the dynamic budget updates match the Python mirror bit for bit
double np_pairwise_sum(const double *a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

// dense.tail_rank (linalg.py:89-99 + the certified remainder)
int64_t tail_rank(const std::vector<double> &s, double delta, int64_t m, int64_t n, double rest2) {
  const int64_t ns = (int64_t)s.size();
  if (delta == 0.0) {
    if (ns == 0 || s[0] == 0.0) return 0;
    const double thr = (double)std::max(m, n) * kEpsD * s[0];
    int64_t c = 0;
    for (double x : s) c += x >= thr;
    return c;
  }
  std::vector<double> tails(ns + 1, 0.0);
  double run = 0.0;
  for (int64_t i = ns - 1; i >= 0; --i) {  // np.cumsum(sq[::-1])[::-1]
    run += s[i] * s[i];
    tails[i] = run;
  }
  const double d2 = delta * delta;
  for (int64_t i = 0; i <= ns; ++i) {
    const double t = rest2 != 0.0 ? tails[i] + rest2 : tails[i];
    if (t <= d2) return i;
  }
  return 0;  // np.argmax of an all-False mask
}

double tail_error(const std::vector<double> &s, int64_t rank, double rest2) {
  std::vector<double> sq;
  for (int64_t i = rank; i < (int64_t)s.size(); ++i) sq.push_back(s[i] * s[i]);
  const double tot = np_pairwise_sum(sq.data(), (int64_t)sq.size()) + rest2;
  return sqrt(std::max(tot, 0.0));
}

struct Core {
  // 0 dense, 1 side L, 2 side R, 3 sparse pivot, 4 side R times a carry kept
  // unscattered (sv: K x r0 col-major, ld K; ftt_scatter.cu)
  int kind = 0;
  int64_t r0 = 0, n = 0, r1 = 0;
  double *data = nullptr;
  bool owned = false;  // allocated here (freed when replaced)
  const int64_t *kept = nullptr;
  int64_t K = 0, r_other = 0;
  double *sv = nullptr;
};

// Dense operands at least this large (elements) stay unscattered for the
// low-rank path of the next step (FTT_SCATTER_MIN overrides: tests).
int64_t scatter_min_elems() {
  const char *e = getenv("FTT_SCATTER_MIN");
  return e ? atoll(e) : ((int64_t)1 << 22);
}

struct Driver {
  ftt_ctx *ctx;
  int d, pivot;
  std::vector<Core> cs;
  const ftt_sparse_pivot *sp;
  int policy;  // 0 static, 1 dynamic, 2 fixed
  double delta, left, right;
  const int64_t *targets;
  int interval_ok;
  std::vector<double *> tmp;  // allocated, not yet owned by a core: freed if a step fails

  int alloc(double **p, size_t elems) {
    cudaError_t e = cudaMallocAsync((void **)p, 8 * std::max<size_t>(elems, 1), ctx->stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error("sweep: allocation of %zu doubles failed", elems);
      return FTT_ERR_OOM;
    }
    tmp.push_back(*p);
    return FTT_OK;
  }
  void forget(double *p) {
    for (size_t i = tmp.size(); i-- > 0;)
      if (tmp[i] == p) {
        tmp.erase(tmp.begin() + i);
        return;
      }
  }
  void drop(double *p) {
    forget(p);
    cudaFreeAsync(p, ctx->stream);
  }
  void drop_all() {
    for (double *p : tmp) cudaFreeAsync(p, ctx->stream);
    tmp.clear();
  }
  void release(Core &c) {
    if (c.owned && c.data) cudaFreeAsync(c.data, ctx->stream);
    if (c.sv) drop(c.sv);
    c.sv = nullptr;
    c.data = nullptr;
    c.owned = false;
  }
  void replace(int k, double *data, int64_t r0, int64_t n, int64_t r1) {
    release(cs[k]);
    forget(data);
    Core c;
    c.kind = 0;
    c.r0 = r0;
    c.n = n;
    c.r1 = r1;
    c.data = data;
    c.owned = true;
    cs[k] = c;
  }
  int densify(int k) {
    Core &c = cs[k];
    if (c.kind == 0) return FTT_OK;
    double *buf = nullptr;
    FTT_CHECK(alloc(&buf, (size_t)c.r0 * c.n * c.r1));
    if (c.kind == 3) {
      FTT_CHECK(ftt_pivot_core_scatter(ctx, sp->nnz, sp->fiber_of, sp->pivot_index, sp->values,
                                       sp->t_map, sp->s_map, c.r0, c.n, c.r1, buf, nullptr));
    } else if (c.kind == 4) {
      FTT_CHECK(ftt_scatter_cols(ctx, c.r0, c.K, c.kept, c.sv, c.K, c.n * c.r1, buf));
    } else {
      FTT_CHECK(ftt_side_core_dense(ctx, c.kind == 1 ? 0 : 1, c.kept, c.K, c.n, c.r_other, buf));
    }
    replace(k, buf, c.r0, c.n, c.r1);
    return FTT_OK;
  }

  static int64_t lowrank_k(int64_t min_dim, int64_t hint) {  // dense.lowrank_k
    if (min_dim < 16) return 0;
    int64_t k = hint < 0 ? 32 : std::max<int64_t>(16, 2 * hint + 8);
    k = (k + 7) / 8 * 8;
    if (k > 64) return 0;
    if (k < min_dim && (2 * k <= min_dim || min_dim <= 64)) return k;
    return 0;
  }

  // dense.dev_svd_truncate / pipeline._sparse_first_step: singular values
  // (+ certified remainder) of the step's operand; the factorisation stays
  // in the context for ftt_svd_vectors.
  int values(int k, int64_t m, int64_t n, bool row_major, bool has_delta, double dlt,
             int64_t hint, bool interval, std::vector<double> *s, double *rest2) {
    Core &c = cs[k];
    *rest2 = 0.0;
    if (has_delta && dlt > 0.0) {
      const int64_t kk = lowrank_k(std::min(m, n), hint);
      if (kk) {
        std::vector<double> sv(kk, 0.0);
        double r2 = 0.0;
        int32_t acc = 0;
        if (c.kind == 3) {
          FTT_CHECK(svd_lowrank_sparse(ctx, m, n, sp->nnz, sp->fiber_of, sp->pivot_index,
                                       sp->values, sp->t_map, sp->s_map, c.n, sp->num_fibers,
                                       sp->indptr, kk, dlt * dlt, sv.data(), &r2, &acc));
        } else if (c.kind == 4) {
          ScatterOperand so;
          so.mA = c.r1;
          so.n = c.n;
          so.r = c.r0;
          so.K = c.K;
          so.kept = c.kept;
          so.V = c.sv;
          so.ldv = c.K;
          FTT_CHECK(svd_lowrank_scatter(ctx, &so, kk, dlt * dlt, sv.data(), &r2, &acc));
        } else {
          FTT_CHECK(ftt_svd_lowrank_f64(ctx, m, n, c.data, row_major ? n : m, row_major ? 1 : 0,
                                        kk, dlt * dlt, sv.data(), &r2, &acc));
        }
        bool ok = acc == 2;
        if (!ok && acc == 1 && interval)
          ok = tail_rank(sv, dlt, m, n, 0.0) == tail_rank(sv, dlt, m, n, r2);
        if (ok) {
          *s = sv;
          *rest2 = r2;
          return FTT_OK;
        }
      }
    }
    ctx->fro2_hint = 0.0;
    if (cs[k].kind != 0) FTT_CHECK(densify(k));
    const int64_t mn = std::min(m, n);
    s->assign(std::max<int64_t>(mn, 1), 0.0);
    FTT_CHECK(ftt_svd_f64(ctx, m, n, cs[k].data, row_major ? n : m, row_major ? 1 : 0, s->data()));
    s->resize(mn);
    return FTT_OK;
  }

  // policy.first / policy.second (pipeline._Trunc)
  int64_t decide(bool first, int k, const std::vector<double> &s, int64_t m, int64_t n,
                 double rest2) {
    if (policy == 0) return tail_rank(s, delta, m, n, rest2);
    if (policy == 1) {
      double &budget = first ? right : left;
      const double dl = first ? budget / sqrt((double)(d - 1 - k)) : budget / sqrt((double)k);
      const int64_t r = tail_rank(s, dl, m, n, rest2);
      const double err = tail_error(s, r, rest2);
      budget = sqrt(std::max(budget * budget - err * err, 0.0));
      return r;
    }
    return std::min<int64_t>(first ? targets[k + 1] : targets[k], std::min(m, n));
  }
  bool step_delta(bool first, int k, double *dl) const {
    if (policy == 0) {
      *dl = delta;
      return true;
    }
    if (policy == 1) {
      *dl = first ? right / sqrt((double)(d - 1 - k)) : left / sqrt((double)k);
      return true;
    }
    return false;
  }

  int run(int32_t *zero) {
    *zero = 0;
    ctx->spec_ok = true;
    int64_t hint = -1;
    // ||operand||_F^2 of a step whose operand is a scattered carry S V^T:
    // the retained singular values' squares (V has orthonormal columns)
    double fro2_next = 0.0;
    const int64_t sc_min = scatter_min_elems();
    for (int k = pivot; k < d - 1; ++k) {  // fasttt.py:334-341
      Core &C = cs[k];
      const int64_t r0 = C.r0, n = C.n, r1 = C.r1, m = r0 * n;
      double dl = 0.0;
      const bool hd = step_delta(true, k, &dl);
      std::vector<double> s;
      double rest2 = 0.0;
      if (fro2_next > 0.0) ctx->fro2_hint = fro2_next;
      fro2_next = 0.0;
      ctx->rank_hint = hint > 0 ? hint : 0;
      FTT_CHECK(values(k, m, r1, true, hd, dl, hint, policy == 0 && interval_ok, &s, &rest2));
      ctx->fro2_hint = 0.0;
      ctx->rank_hint = 0;
      const int64_t rank = decide(true, k, s, m, r1, rest2);
      hint = rank;
      if (rank == 0) {
        *zero = 1;
        return FTT_OK;
      }
      double *U = nullptr, *V = nullptr;
      FTT_CHECK(alloc(&U, (size_t)m * rank));
      FTT_CHECK(alloc(&V, (size_t)r1 * rank));
      FTT_CHECK(ftt_svd_vectors(ctx, rank, U, rank, 1, V, r1, 0, 1));  // V: r1 x rank col-major
      replace(k, U, r0, n, rank);
      Core &N = cs[k + 1];
      double *nw = nullptr;
      if (N.kind == 1 || N.kind == 2) {
        if (N.K == r1)
          for (int64_t i = 0; i < rank; ++i) fro2_next += s[i] * s[i];
        // the next step's operand (rank n x r_other): left unscattered when
        // its low-rank path can run on the compact form (ftt_scatter.cu)
        double dn = 0.0;
        const int64_t mn2 = rank * N.n;
        const bool defer = N.kind == 2 && k + 1 < d - 1 && N.K == r1 && mn2 < N.r_other &&
                           mn2 * N.r_other >= sc_min && step_delta(true, k + 1, &dn) && dn > 0.0 &&
                           lowrank_k(mn2, rank) > 0 &&
                           scatter_operand_ok(N.r_other, N.n, rank, N.K);
        if (defer) {
          Core c4 = N;
          c4.kind = 4;
          c4.r0 = rank;
          c4.r1 = N.r_other;
          c4.sv = V;
          c4.data = nullptr;
          c4.owned = false;
          cs[k + 1] = c4;
          continue;  // V lives on as the core's carry
        }
        FTT_CHECK(alloc(&nw, (size_t)rank * N.n * N.r_other));
        FTT_CHECK(ftt_scatter_cols(ctx, rank, N.K, N.kept, V, r1, N.n * N.r_other, nw));
        const int64_t nn = N.n, ro = N.r_other;
        replace(k + 1, nw, rank, nn, ro);
      } else {
        if (N.kind == 3) FTT_CHECK(densify(k + 1));
        const int64_t nn = cs[k + 1].n, c = cs[k + 1].r1;
        FTT_CHECK(alloc(&nw, (size_t)rank * nn * c));
        FTT_CHECK(ftt_dgemm(ctx, 0, 0, nn * c, rank, r1, 1.0, cs[k + 1].data, nn * c, V, r1, 0.0,
                            nw, nn * c));
        replace(k + 1, nw, rank, nn, c);
      }
      drop(V);
    }
    fro2_next = 0.0;
    for (int k = d - 1; k > pivot; --k) {  // fasttt.py:342-347
      FTT_CHECK(densify(k));
      const int64_t r0 = cs[k].r0, n = cs[k].n, r1 = cs[k].r1;
      const int64_t mq = n * r1, q = std::min(mq, r0);
      double *Q = nullptr, *R = nullptr;
      FTT_CHECK(alloc(&Q, (size_t)mq * q));
      FTT_CHECK(alloc(&R, (size_t)q * r0));
      FTT_CHECK(ftt_qr_f64(ctx, mq, r0, cs[k].data, mq, Q, mq, R, q));
      replace(k, Q, q, n, r1);
      FTT_CHECK(densify(k - 1));
      const int64_t a = cs[k - 1].r0, b = cs[k - 1].n, c = cs[k - 1].r1;
      double *Y = nullptr;
      FTT_CHECK(alloc(&Y, (size_t)a * b * q));
      FTT_CHECK(ftt_dgemm(ctx, 0, 0, q, a * b, c, 1.0, R, q, cs[k - 1].data, c, 0.0, Y, q));
      replace(k - 1, Y, a, b, q);
      drop(R);
    }
    for (int k = pivot; k > 0; --k) {  // fasttt.py:348-355
      FTT_CHECK(densify(k));
      const int64_t r0 = cs[k].r0, n = cs[k].n, r1 = cs[k].r1, m = n * r1;
      double dl = 0.0;
      const bool hd = step_delta(false, k, &dl);
      std::vector<double> s;
      double rest2 = 0.0;
      if (fro2_next > 0.0) ctx->fro2_hint = fro2_next;
      fro2_next = 0.0;
      ctx->rank_hint = hint > 0 ? hint : 0;
      FTT_CHECK(values(k, m, r0, false, hd, dl, hint, policy == 0 && interval_ok, &s, &rest2));
      ctx->fro2_hint = 0.0;
      ctx->rank_hint = 0;
      const int64_t rank = decide(false, k, s, m, r0, rest2);
      hint = rank;
      if (rank == 0) {
        *zero = 1;
        return FTT_OK;
      }
      double *U = nullptr, *V = nullptr;
      FTT_CHECK(alloc(&U, (size_t)m * rank));
      FTT_CHECK(alloc(&V, (size_t)r0 * rank));
      FTT_CHECK(ftt_svd_vectors(ctx, rank, U, m, 0, V, rank, 1, 1));  // V: r0 x rank row-major
      replace(k, U, rank, n, r1);
      Core &Pv = cs[k - 1];
      double *nw = nullptr;
      if (Pv.kind == 1 || Pv.kind == 2) {
        if (Pv.K == r0)
          for (int64_t i = 0; i < rank; ++i) fro2_next += s[i] * s[i];
        FTT_CHECK(alloc(&nw, (size_t)Pv.r_other * Pv.n * rank));
        FTT_CHECK(ftt_scatter_rows(ctx, Pv.K, rank, Pv.kept, V, rank, Pv.r_other * Pv.n, nw));
        const int64_t ro = Pv.r_other, nn = Pv.n;
        replace(k - 1, nw, ro, nn, rank);
      } else {
        if (Pv.kind == 3) FTT_CHECK(densify(k - 1));
        const int64_t a = cs[k - 1].r0, b = cs[k - 1].n, c = cs[k - 1].r1;
        FTT_CHECK(alloc(&nw, (size_t)a * b * rank));
        FTT_CHECK(ftt_dgemm(ctx, 0, 0, rank, a * b, c, 1.0, V, rank, cs[k - 1].data, c, 0.0, nw,
                            rank));
        replace(k - 1, nw, a, b, rank);
      }
      drop(V);
    }
    for (int k = 0; k < d; ++k) {
      FTT_CHECK(densify(k));
      if (!cs[k].owned) {  // an input core left untouched: hand back a copy
        double *cp = nullptr;
        const size_t el = (size_t)cs[k].r0 * cs[k].n * cs[k].r1;
        FTT_CHECK(alloc(&cp, el));
        FTT_CUDA(cudaMemcpyAsync(cp, cs[k].data, 8 * el, cudaMemcpyDeviceToDevice, ctx->stream));
        replace(k, cp, cs[k].r0, cs[k].n, cs[k].r1);
      }
    }
    return FTT_OK;
  }
};

}  // namespace
}  // namespace ftt

using namespace ftt;

extern "C" {

int ftt_free_device(ftt_ctx *ctx, void *p) {
  if (!ctx) return FTT_ERR_INVALID;
  if (p) FTT_CUDA(cudaFreeAsync(p, ctx->stream));
  return FTT_OK;
}

int ftt_sweep_rounding(ftt_ctx *ctx, int32_t d, int32_t pivot, const ftt_core_desc *cores,
                       const ftt_sparse_pivot *sp, int32_t policy, double delta, double left,
                       double right, const int64_t *targets, int32_t interval_ok,
                       double **out_ptrs, int64_t *out_shapes, int32_t *zero_out) {
  if (!ctx || !cores || !out_ptrs || !out_shapes || !zero_out || d < 2 || d > 64 || pivot < 0 ||
      pivot >= d || policy < 0 || policy > 2 || (policy == 2 && !targets)) {
    set_error("ftt_sweep_rounding: invalid arguments");
    return FTT_ERR_INVALID;
  }
  Driver dr;
  dr.ctx = ctx;
  dr.d = d;
  dr.pivot = pivot;
  dr.sp = sp;
  dr.policy = policy;
  dr.delta = delta;
  dr.left = left;
  dr.right = right;
  dr.targets = targets;
  dr.interval_ok = interval_ok;
  dr.cs.resize(d);
  for (int k = 0; k < d; ++k) {
    Core &c = dr.cs[k];
    c.kind = cores[k].kind;
    c.r0 = cores[k].r0;
    c.n = cores[k].n;
    c.r1 = cores[k].r1;
    c.data = cores[k].data;
    c.kept = cores[k].kept;
    c.K = cores[k].K;
    c.r_other = cores[k].r_other;
    if (c.kind == 3 && !sp) {
      set_error("ftt_sweep_rounding: sparse pivot core without entries");
      return FTT_ERR_INVALID;
    }
  }
  int32_t zero = 0;
  const int rc = dr.run(&zero);
  if (rc != FTT_OK || zero) {
    for (auto &c : dr.cs) dr.release(c);
    dr.drop_all();
    *zero_out = zero;
    for (int k = 0; k < d; ++k) out_ptrs[k] = nullptr;
    return rc;
  }
  *zero_out = 0;
  for (int k = 0; k < d; ++k) {
    out_ptrs[k] = dr.cs[k].data;
    out_shapes[3 * k] = dr.cs[k].r0;
    out_shapes[3 * k + 1] = dr.cs[k].n;
    out_shapes[3 * k + 2] = dr.cs[k].r1;
  }
  return FTT_OK;
}

}  // extern "C"
