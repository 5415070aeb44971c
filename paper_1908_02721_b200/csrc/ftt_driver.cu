// fasttt() in one native call (fasttt.py:634-749): select_p, fiber
// extraction, deparallelisation sweeps, the structured train, the rounding
// sweeps and the report's inner-product terms run back to back on the
// context's stream, so the GPU never waits for the Python orchestration
// between the stages (config 2: ~1 ms of host gaps per 2.4 ms decomposition).
// Same kernels, same order and the same host arithmetic as the step-by-step
// path in pipeline.py (which stays as the fallback and as the cross-check:
// tests/test_gpu_parity.py compares the two bit for bit).
#include <math.h>

#include <algorithm>
#include <vector>

#include "ftt_common.cuh"

using namespace ftt;

namespace {

typedef unsigned __int128 u128;

// pipeline.select_p's exact-int cost model (fasttt.py:456-558): bond bounds
// from the fiber count, feasibility caps, then flops_fasttt's three sums.
// Every term is < 2^121 (counts < 2^30, extents < 2^31), so 128-bit integers
// are exact; the cost compared is c_svd * float(total) like the reference.
int pick_pivot(int d, const int64_t *dims, const int64_t *counts, double c_svd) {
  std::vector<int64_t> pre(d + 1, 1), outer(d + 1, 1);
  for (int k = 0; k < d; ++k) pre[k + 1] = pre[k] * dims[k];
  const int64_t size = pre[d];
  for (int k = 0; k <= d; ++k) outer[k] = size / pre[k];
  std::vector<int64_t> caps(d + 1, 1);
  for (int k = 1; k < d; ++k) caps[k] = std::min(pre[k], outer[k]);
  int best = 0;
  double best_cost = INFINITY;
  std::vector<int64_t> rt(d + 1), r(d + 1);
  for (int p = 0; p < d; ++p) {
    const int64_t R = counts[p];
    rt[0] = rt[d] = r[0] = r[d] = 1;
    for (int k = 1; k < d; ++k) {
      rt[k] = k <= p ? std::min(R, pre[k]) : std::min(R, outer[k]);
      r[k] = std::min(rt[k], caps[k]);
    }
    const int p1 = p + 1;
    auto term = [](int64_t m, int64_t n) { return (u128)m * (u128)n * (u128)std::min(m, n); };
    u128 total = term(rt[p1 - 1] * dims[p1 - 1], rt[p1]);
    for (int i = p1 + 1; i < d; ++i) total += term(r[i - 1] * dims[i - 1], rt[i]);
    for (int i = 2; i <= p1; ++i) total += term(rt[i - 1], dims[i - 1] * r[i]);
    const double cost = c_svd * (double)total;
    if (cost < best_cost) {
      best_cost = cost;
      best = p;
    }
  }
  return best;
}

// The output train into one slab: block (x, k) copies a stride of core k.
struct PackSrc {
  const double *src[32];
  int64_t off[33];
};
__global__ void k_pack_cores(PackSrc p, double *__restrict__ slab) {
  const int k = blockIdx.y;
  const int64_t n = p.off[k + 1] - p.off[k];
  const double *__restrict__ s = p.src[k];
  double *__restrict__ d = slab + p.off[k];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

struct Bufs {  // device buffers of one call, released on an error return
  ftt_ctx *ctx;
  std::vector<void *> v;
  void adopt(void *p) {
    if (p) v.push_back(p);
  }
  void forget(void *p) {
    auto it = std::find(v.begin(), v.end(), p);
    if (it != v.end()) v.erase(it);
  }
  int alloc(void **p, size_t bytes) {
    cudaError_t e = cudaMallocAsync(p, std::max<size_t>(bytes, 8), ctx->stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error("fasttt: allocation of %zu bytes failed", bytes);
      return FTT_ERR_OOM;
    }
    v.push_back(*p);
    return FTT_OK;
  }
  void drop_all() {
    for (void *p : v) cudaFreeAsync(p, ctx->stream);
    v.clear();
  }
};

int run(ftt_ctx *ctx, const int64_t *lin, const double *values, int64_t nnz, int32_t d,
        const int64_t *dims, int32_t pivot_in, int32_t mode, double eps, double c_svd,
        int32_t report, void *values_ready, ftt_fasttt_result *res, Bufs &bufs) {
  // ---- select_p (fasttt.py:501-558)
  int pivot = pivot_in;
  if (pivot < 0) {
    int64_t counts[32];
    FTT_CHECK(ftt_fiber_counts_lin(ctx, lin, nullptr, nnz, d, dims, counts));
    pivot = pick_pivot(d, dims, counts, c_svd);
  }
  res->pivot = pivot;
  // the values are first read by the fiber emit: the extraction waits for
  // their upload there, after the key sort (which reads only lin)
  ctx->values_event = (cudaEvent_t)values_ready;
  // ---- fibers (tensor.py:374-403)
  int64_t *fixed_lin, *indptr, *fiber_of, *pidx;
  double *vals;
  {
    void *slab = nullptr;  // one allocation: 4 index arrays + values
    const size_t n8 = 8 * (size_t)nnz;
    FTT_CHECK(bufs.alloc(&slab, 5 * n8 + 8 + 256));
    fixed_lin = (int64_t *)slab;
    indptr = fixed_lin + nnz;  // nnz + 1 entries
    fiber_of = indptr + nnz + 1;
    pidx = fiber_of + nnz;
    vals = (double *)(pidx + nnz);
    res->fiber_slab = slab;
  }
  int64_t R = 0;
  FTT_CHECK(ftt_extract_fibers_lin(ctx, lin, values, nnz, d, dims, pivot, fixed_lin, indptr,
                                   fiber_of, pidx, vals, &R));
  if (ctx->values_event) {  // (a path that did not reach the emit)
    FTT_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->values_event, 0));
    ctx->values_event = nullptr;
  }
  res->num_fibers = R;
  res->fixed_lin = fixed_lin;
  res->indptr = indptr;
  res->fiber_of = fiber_of;
  res->pivot_index = pidx;
  res->values_f = vals;
  // ---- index sweeps (fasttt.py:181-211)
  const int nsteps = d - 1;
  std::vector<int> step_mode(nsteps);
  std::vector<int64_t> ksz(nsteps);
  {
    int s = 0;
    u128 prod = 1;
    for (int k = 0; k < pivot; ++k, ++s) {
      step_mode[s] = k;
      const u128 b = std::min<u128>((u128)R, prod) * (u128)dims[k];
      if (b > (u128)2147483647) return res->fallback = 1, FTT_OK;
      ksz[s] = std::max<int64_t>(std::min<int64_t>(R, (int64_t)b), 1);
      prod *= (u128)dims[k];
    }
    prod = 1;
    for (int k = d - 1; k > pivot; --k, ++s) {
      step_mode[s] = k;
      const u128 b = std::min<u128>((u128)R, prod) * (u128)dims[k];
      if (b > (u128)2147483647) return res->fallback = 1, FTT_OK;
      ksz[s] = std::max<int64_t>(std::min<int64_t>(R, (int64_t)b), 1);
      prod *= (u128)dims[k];
    }
  }
  int64_t ktot = 0;
  for (int s = 0; s < nsteps; ++s) ktot += ksz[s];
  int64_t *kbuf = nullptr, *mbuf = nullptr;
  FTT_CHECK(bufs.alloc((void **)&kbuf, 8 * (size_t)ktot));
  FTT_CHECK(bufs.alloc((void **)&mbuf, 8 * (size_t)std::max<int64_t>(R, 1) * nsteps));
  res->kept_slab = kbuf;
  res->maps_slab = mbuf;
  int64_t *kept[32], *maps[32];
  {
    int64_t off = 0;
    for (int s = 0; s < nsteps; ++s) {
      kept[s] = kbuf + off;
      maps[s] = mbuf + (int64_t)s * std::max<int64_t>(R, 1);
      res->kept_off[s] = off;
      off += ksz[s];
    }
  }
  int64_t *cnt = res->step_counts;
  FTT_CHECK(ftt_index_sweeps_all(ctx, fixed_lin, R, d, dims, pivot, kept, maps, cnt));
  const int64_t *t_map = pivot > 0 ? maps[pivot - 1] : nullptr;
  const int64_t *s_map = pivot < d - 1 ? maps[nsteps - 1] : nullptr;
  const int64_t r_prev = pivot > 0 ? cnt[pivot - 1] : 1;
  const int64_t r_next = pivot < d - 1 ? cnt[nsteps - 1] : 1;
  // ---- ||a||^2 of the report (fasttt.py:596-599)
  double na2 = 0.0;
  if (report) FTT_CHECK(ftt_dot(ctx, nnz, values, nullptr, &na2));
  // ---- structured train (fasttt.py:228-261): 0/1 cores stay index maps
  std::vector<ftt_core_desc> descs(d);
  for (int s = 0; s < nsteps; ++s) {
    const int k = step_mode[s];
    ftt_core_desc &c = descs[k];
    memset(&c, 0, sizeof(c));
    const bool left = k < pivot;
    const bool first = s == 0 || (step_mode[s - 1] < pivot) != left;
    const int64_t r_other = first ? 1 : cnt[s - 1];
    c.kind = left ? 1 : 2;
    c.kept = kept[s];
    c.K = cnt[s];
    c.r_other = r_other;
    c.n = dims[k];
    c.r0 = left ? r_other : cnt[s];
    c.r1 = left ? cnt[s] : r_other;
  }
  const int64_t np = dims[pivot];
  res->pivot_shape[0] = r_prev;
  res->pivot_shape[1] = np;
  res->pivot_shape[2] = r_next;
  ftt_core_desc &pc = descs[pivot];
  memset(&pc, 0, sizeof(pc));
  pc.r0 = r_prev;
  pc.n = np;
  pc.r1 = r_next;
  const u128 pelems = (u128)r_prev * (u128)np * (u128)r_next;
  const double density = (double)nnz / (double)std::max<u128>(pelems, 1);
  ftt_sparse_pivot sp{nnz, fiber_of, pidx, vals, t_map, s_map, R, indptr};
  double pnorm = 0.0;
  double *pdense = nullptr;
  if (density < 0.02 && pivot < d - 1) {  // pipeline._SPARSE_PIVOT_DENSITY
    pc.kind = 3;
    res->lazy_pivot = 1;
    if (!report) FTT_CHECK(ftt_dot(ctx, nnz, vals, nullptr, &na2));
    pnorm = sqrt(na2);
  } else {
    if (pelems > ((u128)1 << 40)) {
      set_error("pivot core (%lld, %lld, %lld) does not fit in device memory", (long long)r_prev,
                (long long)np, (long long)r_next);
      return FTT_ERR_OOM;
    }
    if (bufs.alloc((void **)&pdense, 8 * (size_t)pelems) != FTT_OK) {
      set_error("pivot core (%lld, %lld, %lld) does not fit in device memory", (long long)r_prev,
                (long long)np, (long long)r_next);
      return FTT_ERR_OOM;
    }
    FTT_CHECK(ftt_pivot_core_scatter(ctx, nnz, fiber_of, pidx, vals, t_map, s_map, r_prev, np,
                                     r_next, pdense, &pnorm));
    pc.kind = 0;
    pc.data = pdense;
  }
  res->na2 = na2;
  res->pnorm = pnorm;
  // ---- budget (fasttt.py:364-428)
  const double denom = sqrt((double)pivot) + sqrt((double)(d - 1 - pivot));
  double delta = 0.0, left = 0.0, right = 0.0;
  if (mode == 0) {
    delta = denom != 0.0 ? eps * pnorm / denom : 0.0;
  } else {
    right = denom != 0.0 ? sqrt((double)(d - 1 - pivot)) / denom * eps * pnorm : 0.0;
    left = denom != 0.0 ? sqrt((double)pivot) / denom * eps * pnorm : 0.0;
  }
  // ---- rounding sweeps (fasttt.py:324-356); the sparse first step's
  // operand norm is ||a||^2, already on the host
  if (pc.kind == 3 && na2 > 0.0) ctx->fro2_hint = na2;
  double *out[32];
  int32_t zero = 0;
  FTT_CHECK(ftt_sweep_rounding(ctx, d, pivot, descs.data(), &sp, mode, delta, left, right, nullptr,
                               mode == 0 ? 1 : 0, out, res->out_shapes, &zero));
  if (pdense) {
    cudaFreeAsync(pdense, ctx->stream);
    bufs.forget(pdense);
  }
  res->zero = zero;
  if (!zero)
    for (int k = 0; k < d; ++k) bufs.adopt(out[k]);
  // small trains leave in one slab (one D2H for the caller), large ones as
  // the sweep's own buffers
  int64_t total = 0;
  if (zero) {
    for (int k = 0; k < d; ++k) {
      res->out_shapes[3 * k] = 1;
      res->out_shapes[3 * k + 1] = dims[k];
      res->out_shapes[3 * k + 2] = 1;
      out[k] = nullptr;
    }
  }
  for (int k = 0; k < d; ++k)
    total += res->out_shapes[3 * k] * res->out_shapes[3 * k + 1] * res->out_shapes[3 * k + 2];
  res->out_total = total;
  if (zero || 8 * total <= ((int64_t)16 << 20)) {
    double *slab = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&slab, 8 * (size_t)std::max<int64_t>(total, 1),
                                    ctx->stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error("fasttt: allocation of the output train failed");
      return FTT_ERR_OOM;
    }
    bufs.adopt(slab);
    PackSrc ps;
    int64_t off = 0, widest = 1;
    for (int k = 0; k < d; ++k) {
      const int64_t el =
          res->out_shapes[3 * k] * res->out_shapes[3 * k + 1] * res->out_shapes[3 * k + 2];
      ps.src[k] = out[k];
      ps.off[k] = off;
      widest = std::max(widest, el);
      off += el;
    }
    ps.off[d] = off;
    if (zero) {
      FTT_CUDA(cudaMemsetAsync(slab, 0, 8 * (size_t)std::max<int64_t>(total, 1), ctx->stream));
    } else {  // one launch for all d cores
      k_pack_cores<<<dim3((unsigned)std::min<int64_t>(ceil_div(widest, 1024), 64), (unsigned)d), 256,
                     0, ctx->stream>>>(ps, slab);
      FTT_LAUNCHED(ctx);
    }
    for (int k = 0; k < d; ++k) {
      if (!zero) {
        cudaFreeAsync(out[k], ctx->stream);
        bufs.forget(out[k]);
      }
      out[k] = slab + ps.off[k];
    }
    res->out_slab = slab;
  }
  for (int k = 0; k < d; ++k) res->out_cores[k] = out[k];
  // ---- report terms (fasttt.py:587-602 on the fiber structure)
  if (report) {
    int64_t ranks[33], oc[32];
    ranks[0] = 1;
    for (int k = 0; k < d; ++k) ranks[k + 1] = res->out_shapes[3 * k + 2];
    for (int s = 0; s < nsteps; ++s) oc[s] = cnt[s];
    const int p = pivot;
    u128 cost = 0;
    for (int k = 0; k < p; ++k) cost += (u128)cnt[k] * (u128)ranks[k] * (u128)ranks[k + 1];
    cost += (u128)(p > 0 ? cnt[p - 1] : 1) * (u128)dims[p] * (u128)ranks[p] * (u128)ranks[p + 1];
    for (int q = 0; q < d - 1 - p; ++q)
      cost += (u128)cnt[p + q] * (u128)ranks[d - 1 - q] * (u128)ranks[d - q];
    if (cost <= (u128)4000000000ull && na2 != 0.0) {
      const double *cp[32];
      for (int k = 0; k < d; ++k) cp[k] = out[k];
      const int64_t *kp[32];
      for (int s = 0; s < nsteps; ++s) kp[s] = kept[s];
      FTT_CHECK(ftt_inner_structured(ctx, d, dims, ranks, cp, pivot, kp, oc, R, indptr, pidx, vals,
                                     t_map, s_map, &res->dot));
      // ||b||: the sweeps leave cores 1..d-1 right-orthogonal (QR sweep, then
      // the V factors of the second SVD sweep), so the train's norm is core
      // 0's (fasttt.py:598 computes tt_norm of the same train)
      double nb2 = 0.0;
      FTT_CHECK(ftt_dot(ctx, res->out_shapes[0] * res->out_shapes[1] * res->out_shapes[2], out[0],
                        nullptr, &nb2));
      res->nb = sqrt(nb2);
      res->inner_valid = 1;
    }
  }
  return FTT_OK;
}

}  // namespace

extern "C" {

int ftt_fasttt_lin(ftt_ctx *ctx, const int64_t *lin, const double *values, int64_t nnz, int32_t d,
                   const int64_t *dims, int32_t pivot, int32_t mode, double eps, double c_svd,
                   int32_t report, void *values_ready, ftt_fasttt_result *res) {
  if (!ctx || !lin || !values || !dims || !res || nnz < 1 || d < 2 || d > 32 || pivot >= d ||
      mode < 0 || mode > 1) {
    if (ctx) {  // a chunk list set for this call does not outlive it
      ctx->lin_nchunks = 0;
      ctx->values_event = nullptr;
    }
    set_error("ftt_fasttt_lin: invalid arguments");
    return FTT_ERR_INVALID;
  }
  memset(res, 0, sizeof(*res));
  struct ChunkWait {  // a chunked lin upload nobody consumed: the stream waits for it
    ftt_ctx *c;
    ~ChunkWait() {
      lin_chunks_wait_all(c);
      c->values_event = nullptr;  // (an error return before the emit)
    }
  } chunk_wait{ctx};
  for (int k = 0; k < d; ++k)
    if (dims[k] < 1 || dims[k] >= ((int64_t)1 << 31)) return res->fallback = 1, FTT_OK;
  if (nnz >= ((int64_t)1 << 30)) return res->fallback = 1, FTT_OK;
  Bufs bufs{ctx, {}};
  const bool deferred = ctx->defer_checks;
  ctx->defer_checks = true;
  int rc = run(ctx, lin, values, nnz, d, dims, pivot, mode, eps, c_svd, report, values_ready, res,
               bufs);
  ctx->defer_checks = deferred;
  int32_t flags = 0;
  const int rs = ftt_take_status(ctx, &flags);
  if (rc == FTT_OK) rc = rs;
  res->status_flags = flags;
  if (rc != FTT_OK || res->fallback) {
    bufs.drop_all();
    res->fiber_slab = res->kept_slab = res->maps_slab = nullptr;
    res->out_slab = nullptr;
    for (int k = 0; k < d; ++k) res->out_cores[k] = nullptr;
  }
  return rc;
}

}  // extern "C"
