"""FastTT on one B200: the drop-in for the reference ``fasttt.py`` hot path.

Stages (reference fasttt.py:634-749) and where they run:

1. ``select_p`` -- per-pivot fiber counts from one device radix sort per mode
   (``ftt_fiber_counts_all``); the SVD cost model stays in exact Python ints
   (fasttt.py:456-481, 501-558) because it is a scalar recurrence over d.
2. ``build_structured_tt`` -- ``ftt_extract_fibers`` (sort + segment).
3. ``parallel_vector_round`` -- ``ftt_index_sweep_step`` per mode
   (deparallelisation by flags + scan, bit-exact ascending ranks); only the
   pivot core is materialised (``ftt_pivot_core_scatter``); the 0/1 side
   cores stay as ``kept`` index arrays.
4. rounding -- the three sweeps of _sweep_rounding (fasttt.py:324-356) with
   the device SVD/QR; carries into 0/1 cores are scatters
   (``ftt_scatter_cols`` / ``ftt_scatter_rows``), dense carries DMMA GEMMs.
5. report -- norms, ``tt_entries`` and the capped TT-difference measure on the
   device.

The Python here is orchestration: shapes, ranks, budgets and the choice of
kernel. All arrays on the path are device tensors.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .coo import (
    ContractViolationError,
    FiberSet,
    SparseTensor,
    check_shape,
    device_dot,
    fibers_device,
)
from .dense import (
    dev_svd_truncate,
    dev_svd_values,
    dev_svd_vectors,
    lowrank_k,
    tail_error,
    tail_rank,
)
from .trains import (
    QuasiPermMatrix,
    StructuredTT,
    TTTensor,
    dev_right_orthogonalize,
    dev_tt_entries,
    dev_tt_norm,
    dgemm,
    dev_qr,
    to_device,
    tt_zero,
)

__all__ = [
    "float_ops",
    "TruncationBudget",
    "DecompositionReport",
    "depar_quasi_perm",
    "depar_general",
    "build_structured_tt",
    "parallel_vector_round",
    "efficient_tt_rounding",
    "dynamic_tt_rounding",
    "fixed_rank_rounding",
    "fasttt",
    "fasttt_device",
    "flops_fasttt",
    "flops_ttsvd",
    "full_ranks",
    "select_p",
    "tt_relative_error",
    "sparse_inner_error",
]

_MODES = ("static", "dynamic", "fixed_rank")
_ERROR_MEASURE_CAP = 20_000_000  # fasttt.py:74
# FTT_STEPWISE=1: orchestrate the stages from Python (the fallback path) even
# where the fused native driver applies -- the cross-check of the two
_STEPWISE = __import__("os").environ.get("FTT_STEPWISE") == "1"


class _FlopCounter:
    """Floating-point work issued by deparallelisation (fasttt.py:77-93).
    The index-only routes here never add to it."""

    __slots__ = ("count",)

    def __init__(self):
        self.count = 0.0

    def add(self, n: float) -> None:
        self.count += float(n)

    def reset(self) -> None:
        self.count = 0.0


float_ops = _FlopCounter()


def _torch():
    return nat.torch_mod()


def _empty(shape, dtype="f64"):
    torch = _torch()
    dt = torch.float64 if dtype == "f64" else torch.int64
    return torch.empty(shape, dtype=dt, device="cuda")


# ------------------------------------------------------------ cost model
def full_ranks(shape, ranks) -> tuple[int, ...]:
    """Interior (d-1) or full (d+1) rank vector -> full vector (ttsvd.py:79-98)."""
    dims = check_shape(shape)
    d = len(dims)
    rk = tuple(int(r) for r in ranks)
    if len(rk) == d - 1:
        rk = (1,) + rk + (1,)
    if len(rk) != d + 1:
        raise ValueError(f"rank vector must have length {d - 1} or {d + 1}, got {len(rk)}")
    if rk[0] != 1 or rk[-1] != 1:
        raise ValueError("edge ranks must be 1")
    if any(r < 0 for r in rk):
        raise ValueError("ranks must be nonnegative")
    return rk


def flops_ttsvd(shape, ranks, c_svd: float = 1.0) -> float:
    """Cost model of classical TT-SVD (ttsvd.py:101-116)."""
    dims = check_shape(shape)
    r = full_ranks(dims, ranks)
    total = 0
    for k in range(1, len(dims)):
        rows = r[k - 1] * dims[k - 1]
        cols = math.prod(dims[k:])
        total += rows * cols * min(rows, cols)
    return c_svd * float(total)


def _check_pivot(pivot: int, d: int) -> None:
    if not 0 <= pivot < d:
        raise ValueError(f"pivot {pivot} out of range for {d} modes")


def flops_fasttt(shape, pivot: int, ranks_lossless, ranks_final, c_svd: float = 1.0) -> float:
    """SVD cost model of the pipeline at one pivot (fasttt.py:456-481):
    an m x n SVD costs ``c_svd * m * n * min(m, n)``, summed in exact ints."""
    dims = check_shape(shape)
    d = len(dims)
    _check_pivot(pivot, d)
    if d == 1:
        return 0.0
    return _flops_core(dims, pivot, full_ranks(dims, ranks_lossless), full_ranks(dims, ranks_final),
                       c_svd)


def _flops_core(dims, pivot, rt, r, c_svd):
    """flops_fasttt on validated full rank vectors (select_p's inner loop)."""
    d = len(dims)
    p1 = pivot + 1

    def cost(m, n):
        return m * n * min(m, n)

    total = cost(rt[p1 - 1] * dims[p1 - 1], rt[p1])
    for i in range(p1 + 1, d):
        total += cost(r[i - 1] * dims[i - 1], rt[i])
    for i in range(2, p1 + 1):
        total += cost(rt[i - 1], dims[i - 1] * r[i])
    return c_svd * float(total)


def _upper_bond_bounds(dims, pivot: int, num_fibers: int):
    """Lossless-rank bound per bond (fasttt.py:484-498)."""
    d = len(dims)
    pre = [1]
    for n in dims:
        pre.append(pre[-1] * n)
    size = pre[d]
    return tuple(min(num_fibers, pre[k]) if k < pivot + 1 else min(num_fibers, size // pre[k])
                 for k in range(1, d))


def _fiber_counts_device(a: SparseTensor):
    if a.nnz == 0:
        return [0] * a.ndim
    # the coordinate rows serve only the overflow fallback: passed when the
    # tensor already holds them, else the native side rebuilds them from lin
    c = a._dev[0] if a._dev is not None else None
    counts = (nat.ctypes.c_int64 * a.ndim)()
    nat.check(nat.lib().ftt_fiber_counts_lin(nat.context(), nat.ptr(a.device_lin()), nat.ptr(c),
                                             a.nnz, a.ndim, nat.i64_array(a.shape), counts),
              "ftt_fiber_counts_lin")
    return [int(x) for x in counts]


def select_p(a: SparseTensor, target_ranks=None, precise: bool = False, c_svd: float = 1.0) -> int:
    """Pivot with the smallest modelled SVD cost; ties -> smaller mode
    (fasttt.py:501-558). Fiber counts come from the device."""
    if not isinstance(a, SparseTensor):
        raise TypeError("select_p expects a SparseTensor")
    d = a.ndim
    if d == 1:
        return 0
    dims = a.shape
    pre = [1]
    for n in dims:
        pre.append(pre[-1] * n)
    size = pre[d]
    if target_ranks is None:
        targets = None
    elif isinstance(target_ranks, (int, np.integer)):
        targets = (int(target_ranks),) * (d - 1)
    else:
        targets = tuple(int(r) for r in target_ranks)
        if len(targets) != d - 1:
            raise ValueError(f"need {d - 1} interior rank targets")
    counts = _fiber_counts_device(a) if not precise else None
    # exact-int cost model (fasttt.py:456-558) in one tight loop: bounds of
    # _upper_bond_bounds, feasibility caps, then flops_fasttt's three sums
    outer = [size // pre[k] for k in range(d + 1)]
    caps = [min(pre[k], outer[k]) for k in range(1, d)]
    if targets is not None:
        caps = [min(c, t) for c, t in zip(caps, targets)]
    best_pivot, best_cost = 0, math.inf
    for pivot in range(d):
        if precise:
            rt = list(_lossless_bond_ranks(build_structured_tt(a, pivot)))
        else:
            R = counts[pivot]
            rt = [min(R, pre[k]) if k <= pivot else min(R, outer[k]) for k in range(1, d)]
        r = [1] + [min(x, c) for x, c in zip(rt, caps)] + [1]
        rt = [1] + rt + [1]
        p1 = pivot + 1
        m, n = rt[p1 - 1] * dims[p1 - 1], rt[p1]
        total = m * n * (m if m < n else n)
        for i in range(p1 + 1, d):
            m, n = r[i - 1] * dims[i - 1], rt[i]
            total += m * n * (m if m < n else n)
        for i in range(2, p1 + 1):
            m, n = rt[i - 1], dims[i - 1] * r[i]
            total += m * n * (m if m < n else n)
        cost = c_svd * float(total)
        if cost < best_cost:
            best_cost, best_pivot = cost, pivot
    return best_pivot


# ------------------------------------------------------------ index path
class SideCore:
    """A 0/1 core kept as its index map (never densified on the hot path).

    kind 'L' (left of pivot): shape (r_other, n, K), 1 at [kept//n, kept%n, j]
    kind 'R' (right of pivot): shape (K, n, r_other), 1 at [j, kept//r, kept%r]
    """

    __slots__ = ("kind", "kept", "r_other", "n")

    def __init__(self, kind, kept, r_other, n):
        self.kind = kind
        self.kept = kept
        self.r_other = int(r_other)
        self.n = int(n)

    @property
    def K(self) -> int:
        return int(self.kept.shape[0])

    @property
    def shape(self):
        if self.kind == "L":
            return (self.r_other, self.n, self.K)
        return (self.K, self.n, self.r_other)

    def dense(self):
        core = _empty(self.shape)
        nat.check(nat.lib().ftt_side_core_dense(nat.context(), 0 if self.kind == "L" else 1,
                                                nat.ptr(self.kept), self.K, self.n, self.r_other,
                                                nat.ptr(core)), "ftt_side_core_dense")
        return core


class DeviceSweeps:
    __slots__ = ("left", "t_map", "r_prev", "right", "s_map", "r_next")

    def __init__(self, left, t_map, r_prev, right, s_map, r_next):
        self.left = left
        self.t_map = t_map
        self.r_prev = r_prev
        self.right = right
        self.s_map = s_map
        self.r_next = r_next


def _index_sweeps_batched(df):
    """All sweep steps in one native call (ftt_index_sweeps_all, one host
    round trip); None when a step's flag bound is too large for it."""
    dims, p, R = df.dims, df.pivot, df.R
    d = len(dims)
    steps = list(range(p)) + list(range(d - 1, p, -1))
    bounds, prod_l, prod_r = [], 1, 1
    for k in steps:
        if k < p:
            bounds.append(min(R, prod_l) * dims[k])
            prod_l *= dims[k]
        else:
            bounds.append(min(R, prod_r) * dims[k])
            prod_r *= dims[k]
    if any(b > 2 ** 31 - 1 for b in bounds):
        return None
    # one allocation each for every step's kept rows and maps (views)
    ksz = [max(min(R, b), 1) for b in bounds]
    kbuf = _empty(sum(ksz), "i64")
    mbuf = _empty(max(R, 1) * len(steps), "i64")
    offs = np.cumsum([0] + ksz)
    kept = [kbuf[offs[i]:offs[i + 1]] for i in range(len(steps))]
    maps = [mbuf[i * max(R, 1):(i + 1) * max(R, 1)] for i in range(len(steps))]
    base_k, base_m = kbuf.data_ptr(), mbuf.data_ptr()
    kp = (nat.ctypes.c_void_p * len(steps))(*[base_k + 8 * int(offs[i]) for i in range(len(steps))])
    mp = (nat.ctypes.c_void_p * len(steps))(*[base_m + 8 * i * max(R, 1) for i in range(len(steps))])
    counts = (nat.ctypes.c_int64 * len(steps))()
    nat.check(nat.lib().ftt_index_sweeps_all(nat.context(), nat.ptr(df.fixed_lin), R, d,
                                              nat.i64_array(dims), p, kp, mp, counts),
              "ftt_index_sweeps_all")
    left, right = [], []
    t_map, r_prev, s_map, r_next = None, 1, None, 1
    for i, k in enumerate(steps):
        n = int(counts[i])
        if k < p:
            left.append((kept[i][:n], r_prev))
            t_map, r_prev = maps[i][:R], n
        else:
            right.append((kept[i][:n], r_next))
            s_map, r_next = maps[i][:R], n
    return DeviceSweeps(left, t_map, r_prev, right, s_map, r_next)


def index_sweeps_device(df) -> DeviceSweeps:
    """_index_sweeps (fasttt.py:181-211): every step in one native call when
    the flag bounds allow, else one fused kernel chain per mode."""
    dims, p, R = df.dims, df.pivot, df.R
    d = len(dims)
    if R > 0 and d > 1:
        sw = _index_sweeps_batched(df)
        if sw is not None:
            return sw
    lib, ctx = nat.lib(), nat.context()
    t_map, r_prev, left = None, 1, []
    for k in range(p):
        nk = dims[k]
        kept = _empty(max(min(R, r_prev * nk), 1), "i64")
        mo = _empty(max(R, 1), "i64")
        nkept = nat.ctypes.c_int64(0)
        nat.check(lib.ftt_index_sweep_step(ctx, 0, nat.ptr(df.fixed_lin), R, df.rest_stride(k), nk,
                                           nat.ptr(t_map), r_prev, nat.ptr(kept), nat.ptr(mo),
                                           nat.ctypes.byref(nkept)), "ftt_index_sweep_step")
        left.append((kept[:nkept.value], r_prev))
        t_map, r_prev = mo[:R], int(nkept.value)
    s_map, r_next, right = None, 1, []
    for k in range(d - 1, p, -1):
        nk = dims[k]
        kept = _empty(max(min(R, r_next * nk), 1), "i64")
        mo = _empty(max(R, 1), "i64")
        nkept = nat.ctypes.c_int64(0)
        nat.check(lib.ftt_index_sweep_step(ctx, 1, nat.ptr(df.fixed_lin), R, df.rest_stride(k), nk,
                                           nat.ptr(s_map), r_next, nat.ptr(kept), nat.ptr(mo),
                                           nat.ctypes.byref(nkept)), "ftt_index_sweep_step")
        right.append((kept[:nkept.value], r_next))
        s_map, r_next = mo[:R], int(nkept.value)
    return DeviceSweeps(left, t_map, r_prev, right, s_map, r_next)


def _lossless_ranks_from(sw: DeviceSweeps, d: int):
    bonds = [0] * (d - 1)
    for k, (kept, _) in enumerate(sw.left):
        bonds[k] = int(kept.shape[0])
    for step, (kept, _) in enumerate(sw.right):
        bonds[d - 2 - step] = int(kept.shape[0])
    return tuple(bonds)


def _device_fibers_of(s: StructuredTT):
    f = s.fibers
    if f._dev is not None:
        return f._dev
    # a FiberSet built on the host: upload and rebuild the device view
    from .coo import DeviceFibers

    torch = _torch()
    dims, p = f.shape, f.pivot
    rest = [dims[k] for k in range(len(dims)) if k != p]
    st = np.ones(len(rest), dtype=np.int64)
    for j in range(len(rest) - 2, -1, -1):
        st[j] = st[j + 1] * rest[j + 1]
    fixed_lin = f.fixed_coords @ st if len(rest) else np.zeros(f.num_fibers, np.int64)
    fiber_of = np.repeat(np.arange(f.num_fibers, dtype=np.int64), np.diff(f.indptr))
    return DeviceFibers(tuple(dims), p, f.num_fibers, f.nnz, to_device(fixed_lin.astype(np.int64)),
                        to_device(f.indptr), to_device(fiber_of), to_device(f.pivot_index),
                        to_device(f.values)) if f.num_fibers else DeviceFibers(
        tuple(dims), p, 0, 0, torch.zeros(0, dtype=torch.int64, device="cuda"),
        torch.zeros(1, dtype=torch.int64, device="cuda"),
        torch.zeros(0, dtype=torch.int64, device="cuda"),
        torch.zeros(0, dtype=torch.int64, device="cuda"),
        torch.zeros(0, dtype=torch.float64, device="cuda"))


def _lossless_bond_ranks(s: StructuredTT):
    """_lossless_bond_ranks (fasttt.py:214-225) from the device sweeps."""
    df = _device_fibers_of(s)
    if df.R == 0:
        return (0,) * (s.ndim - 1)
    return _lossless_ranks_from(index_sweeps_device(df), s.ndim)


def depar_general(m, tol: float = 1e-12):
    """Split ``m`` into ``n @ t`` keeping one representative per parallel
    class of columns, in first-occurrence order (fasttt.py:96-145), on the
    GPU (ftt_depar_general).  Column ``u`` is parallel to a kept ``v`` when
    ``norm(u - (u . v_hat) v_hat) <= tol * norm(u)``; zero columns are
    dropped.  Returns dense ``(n, t)`` and counts the same float work as the
    reference into ``float_ops``."""
    import scipy.sparse

    if isinstance(m, QuasiPermMatrix):
        m = m.to_dense()
    elif scipy.sparse.issparse(m):
        m = m.toarray()
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2:
        raise ValueError("deparallelisation expects a matrix")
    rows, cols = m.shape
    if cols == 0:
        return np.zeros((rows, 0)), np.zeros((0, 0))
    torch = _torch()
    md = to_device(np.ascontiguousarray(m.T))  # column-major rows x cols
    kept = torch.empty(cols, dtype=torch.int64, device="cuda")
    t_row = torch.empty(cols, dtype=torch.int64, device="cuda")
    t_coeff = torch.empty(cols, dtype=torch.float64, device="cuda")
    width_at = torch.empty(cols, dtype=torch.int64, device="cuda")
    width = nat.ctypes.c_int64(0)
    nat.check(nat.lib().ftt_depar_general(nat.context(), rows, cols, nat.ptr(md), max(rows, 1),
                                          float(tol), nat.ptr(kept), nat.ptr(t_row),
                                          nat.ptr(t_coeff), nat.ptr(width_at),
                                          nat.ctypes.byref(width)), "ftt_depar_general")
    w = int(width.value)
    kept_h = kept[:w].cpu().numpy()
    t_row_h = t_row.cpu().numpy()
    t_coeff_h = t_coeff.cpu().numpy()
    wat = width_at.cpu().numpy()
    # float work of the reference loop: 2 rows per column norm, 6 rows per
    # tested basis column (fasttt.py:117-127)
    nonzero = t_row_h >= 0
    float_ops.add(float(2 * rows * cols + 6 * rows * int(np.sum(wat[nonzero]))))
    n = np.ascontiguousarray(m[:, kept_h])
    t = np.zeros((w, cols))
    t[t_row_h[nonzero], np.flatnonzero(nonzero)] = t_coeff_h[nonzero]
    return n, t


def depar_quasi_perm(q: QuasiPermMatrix):
    """Deparallelise a quasi-permutation by index arithmetic only
    (fasttt.py:148-167) -- ftt_depar_quasi_perm (flags + scan on the GPU)."""
    if not isinstance(q, QuasiPermMatrix):
        raise TypeError("depar_quasi_perm expects a QuasiPermMatrix")
    if q.n_cols == 0 or q.n_rows == 0:
        kept = np.zeros(0, np.int64)
        return (QuasiPermMatrix(q.n_rows, 0, kept), QuasiPermMatrix(0, q.n_cols, np.zeros(q.n_cols, np.int64)))
    col = to_device(q.col_to_row)
    kept = _empty(min(q.n_rows, q.n_cols), "i64")
    tmap = _empty(q.n_cols, "i64")
    nk = nat.ctypes.c_int64(0)
    nat.check(nat.lib().ftt_depar_quasi_perm(nat.context(), q.n_rows, q.n_cols, nat.ptr(col),
                                             nat.ptr(kept), nat.ptr(tmap), nat.ctypes.byref(nk)),
              "ftt_depar_quasi_perm")
    K = int(nk.value)
    return (QuasiPermMatrix(q.n_rows, K, kept[:K].cpu().numpy()),
            QuasiPermMatrix(K, q.n_cols, tmap.cpu().numpy()))


def build_structured_tt(a: SparseTensor, pivot: int) -> StructuredTT:
    """Exact structured train along ``pivot`` (fasttt.py:170-178)."""
    if not isinstance(a, SparseTensor):
        raise TypeError("build_structured_tt expects a SparseTensor")
    from .coo import extract_nonzero_fibers

    return StructuredTT(extract_nonzero_fibers(a, pivot))


def _pivot_core(df, sw: DeviceSweeps):
    """Dense pivot core + the 2-norm of its values (fasttt.py:256-259, 359-361)."""
    dims, p = df.dims, df.pivot
    shape = (sw.r_prev, dims[p], sw.r_next)
    try:
        core = _empty(shape)
    except RuntimeError as e:  # torch OOM
        raise MemoryError(f"pivot core {shape} does not fit in device memory") from e
    norm = nat.ctypes.c_double(0.0)
    nat.check(nat.lib().ftt_pivot_core_scatter(
        nat.context(), df.nnz, nat.ptr(df.fiber_of), nat.ptr(df.pivot_index), nat.ptr(df.values),
        nat.ptr(sw.t_map), nat.ptr(sw.s_map), sw.r_prev, dims[p], sw.r_next, nat.ptr(core),
        nat.ctypes.byref(norm)), "ftt_pivot_core_scatter")
    return core, float(norm.value)


class SparsePivotCore:
    """The pivot core of parallel_vector_round (fasttt.py:256-259) kept as its
    entries -- value at (t_map[f], i_p, s_map[f]) -- until a dense copy is
    needed.  The first truncation step runs the certified low-rank range
    finder on the entries (ftt_svd_lowrank_sparse_f64); config 5's core is
    0.65 % dense and 10.5 GB when materialised."""

    __slots__ = ("df", "sw", "shape", "_dense")

    def __init__(self, df, sw: DeviceSweeps):
        self.df, self.sw = df, sw
        self.shape = (sw.r_prev, df.dims[df.pivot], sw.r_next)
        self._dense = None

    @property
    def density(self) -> float:
        return self.df.nnz / float(max(math.prod(self.shape), 1))

    def dense(self):
        if self._dense is None:
            self._dense, _ = _pivot_core(self.df, self.sw)
        return self._dense

    def svd_lowrank(self, k: int, delta: float):
        """(s, rest2, accepted) of the first sweep step's operand
        core.reshape(r_prev n_p, r_next) (see dense.dev_svd_values_lowrank)."""
        r0, n, r1 = self.shape
        df, sw = self.df, self.sw
        s = np.zeros(k)
        rest2 = nat.ctypes.c_double(0.0)
        acc = nat.ctypes.c_int32(0)
        nat.check(nat.lib().ftt_svd_lowrank_sparse_f64(
            nat.context(), r0 * n, r1, df.nnz, nat.ptr(df.fiber_of), nat.ptr(df.pivot_index),
            nat.ptr(df.values), nat.ptr(sw.t_map), nat.ptr(sw.s_map), n, int(k),
            float(delta * delta), s.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_double)),
            nat.ctypes.byref(rest2), nat.ctypes.byref(acc)), "ftt_svd_lowrank_sparse_f64")
        return s, float(rest2.value), int(acc.value)


# below this density the first truncation step works on the pivot core's
# entries (sorting them twice costs about as much as one pass over a dense
# core of ~20x the entry count)
_SPARSE_PIVOT_DENSITY = 0.02


def _as_dense(c):
    return c.dense() if isinstance(c, (SideCore, SparsePivotCore)) else c


def _structured_train(df, sw: DeviceSweeps, lazy_pivot: bool = False, na2=None):
    d = len(df.dims)
    cores = [None] * d
    for k, (kept, rp) in enumerate(sw.left):
        cores[k] = SideCore("L", kept, rp, df.dims[k])
    for step, (kept, rn) in enumerate(sw.right):
        k = d - 1 - step
        cores[k] = SideCore("R", kept, rn, df.dims[k])
    if lazy_pivot:
        spc = SparsePivotCore(df, sw)
        if spc.density < _SPARSE_PIVOT_DENSITY and df.pivot < d - 1:
            # ||pivot core||_F = ||values||_2 (fasttt.py:359-361); the caller's
            # sum of squares of the input values when it has one
            cores[df.pivot] = spc
            return cores, math.sqrt(na2 if na2 is not None else device_dot(df.values, None))
    pc, norm = _pivot_core(df, sw)
    cores[df.pivot] = pc
    return cores, norm


def parallel_vector_round(s: StructuredTT) -> TTTensor:
    """Lossless deparallelisation (fasttt.py:228-261). Returns the dense train
    like the reference (the 0/1 cores are materialised only here, for the
    standalone API; fasttt() keeps them as index maps)."""
    if not isinstance(s, StructuredTT):
        raise TypeError("parallel_vector_round expects a StructuredTT")
    if s.num_fibers == 0:
        return tt_zero(s.shape)
    df = _device_fibers_of(s)
    sw = index_sweeps_device(df)
    cores, _ = _structured_train(df, sw)
    out = [_as_dense(c) for c in cores]
    return TTTensor([c.cpu().numpy() for c in out], copy=False)


# -------------------------------------------------------------- rounding
@dataclass(frozen=True)
class TruncationBudget:
    """Error allowance of a rounding pass (fasttt.py:264-295)."""

    eps: float = 1e-14
    pivot: int = 0
    mode: str = "static"
    fixed_ranks: tuple | int | None = None
    delta_left: float | None = None
    delta_right: float | None = None

    def __post_init__(self):
        if self.mode not in _MODES:
            raise ValueError(f"mode must be one of {_MODES}, got {self.mode!r}")
        if self.eps < 0:
            raise ValueError(f"eps must be nonnegative, got {self.eps}")
        if self.pivot < 0:
            raise ValueError(f"pivot must be nonnegative, got {self.pivot}")
        if self.mode == "fixed_rank" and self.fixed_ranks is None:
            raise ValueError("fixed_rank mode needs fixed_ranks")
        for name in ("delta_left", "delta_right"):
            v = getattr(self, name)
            if v is not None and v < 0:
                raise ValueError(f"{name} must be nonnegative")


class _Trunc:
    """Per-step truncation policy (static / dynamic / fixed-rank).

    ``delta_first/second`` give the step's tolerance before the SVD (None in
    fixed-rank mode); ``first/second`` turn the singular values (plus the
    certified remainder ``rest2`` of the low-rank path) into the kept rank and
    update the dynamic budget (fasttt.py:416-426)."""

    def __init__(self, kind, d, delta=0.0, left=0.0, right=0.0, targets=None):
        self.kind, self.d = kind, d
        self.delta, self.left, self.right = delta, left, right
        self.targets = targets

    def delta_first(self, k):
        if self.kind == "static":
            return self.delta
        if self.kind == "dynamic":
            return self.right / math.sqrt(self.d - 1 - k)
        return None

    def delta_second(self, k):
        if self.kind == "static":
            return self.delta
        if self.kind == "dynamic":
            return self.left / math.sqrt(k)
        return None

    def first(self, k, s, shape, rest2=0.0):
        if self.kind == "static":
            r = tail_rank(s, self.delta, shape, rest2)
            return r, tail_error(s, r, rest2)
        if self.kind == "dynamic":
            r = tail_rank(s, self.right / math.sqrt(self.d - 1 - k), shape, rest2)
            err = tail_error(s, r, rest2)
            self.right = math.sqrt(max(self.right ** 2 - err ** 2, 0.0))
            return r, err
        r = int(min(self.targets[k + 1], min(shape)))
        return r, tail_error(s, r)

    def second(self, k, s, shape, rest2=0.0):
        if self.kind == "static":
            r = tail_rank(s, self.delta, shape, rest2)
            return r, tail_error(s, r, rest2)
        if self.kind == "dynamic":
            r = tail_rank(s, self.left / math.sqrt(k), shape, rest2)
            err = tail_error(s, r, rest2)
            self.left = math.sqrt(max(self.left ** 2 - err ** 2, 0.0))
            return r, err
        r = int(min(self.targets[k], min(shape)))
        return r, tail_error(s, r)


class _CoreDesc(nat.ctypes.Structure):
    _fields_ = [("kind", nat.ctypes.c_int32), ("r0", nat.ctypes.c_int64),
                ("n", nat.ctypes.c_int64), ("r1", nat.ctypes.c_int64),
                ("data", nat.ctypes.c_void_p), ("kept", nat.ctypes.c_void_p),
                ("K", nat.ctypes.c_int64), ("r_other", nat.ctypes.c_int64)]


class _SparsePivot(nat.ctypes.Structure):
    _fields_ = [("nnz", nat.ctypes.c_int64), ("fiber_of", nat.ctypes.c_void_p),
                ("pivot_index", nat.ctypes.c_void_p), ("values", nat.ctypes.c_void_p),
                ("t_map", nat.ctypes.c_void_p), ("s_map", nat.ctypes.c_void_p),
                ("num_fibers", nat.ctypes.c_int64), ("indptr", nat.ctypes.c_void_p)]


class _NativeCore:
    """A core buffer allocated by ftt_sweep_rounding, exposed to torch through
    __cuda_array_interface__ (zero copy) and released (ftt_free_device,
    stream-ordered) when the last tensor viewing it is gone."""

    __slots__ = ("ptr", "shape", "typestr", "__weakref__")

    def __init__(self, ptr, shape, typestr="<f8"):
        self.ptr, self.shape, self.typestr = int(ptr), tuple(int(x) for x in shape), typestr

    @property
    def __cuda_array_interface__(self):
        return {"shape": self.shape, "typestr": self.typestr, "data": (self.ptr, False),
                "version": 3, "strides": None}

    def __del__(self):
        try:
            nat.lib().ftt_free_device(nat.context(), nat.ctypes.c_void_p(self.ptr))
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass


def _sweep_rounding_device(cores, pivot: int, policy: _Trunc):
    """_sweep_rounding (fasttt.py:324-356) in one native call
    (ftt_sweep_rounding: the three sweeps and the truncation policy run in
    C++ over the same kernels).  FTT_PY_SWEEP=1 selects the step-by-step
    Python driver below (same kernels, same order)."""
    import os

    if os.environ.get("FTT_PY_SWEEP") == "1":
        return _sweep_rounding_python(cores, pivot, policy)
    torch = _torch()
    d = len(cores)
    descs = (_CoreDesc * d)()
    sp = None
    keep = []  # contiguous copies referenced by the descriptors
    for k, c in enumerate(cores):
        dsc = descs[k]
        if isinstance(c, SideCore):
            dsc.kind = 1 if c.kind == "L" else 2
            dsc.kept, dsc.K, dsc.r_other = c.kept.data_ptr(), c.K, c.r_other
            dsc.r0, dsc.n, dsc.r1 = c.shape
        elif isinstance(c, SparsePivotCore):
            dsc.kind = 3
            dsc.r0, dsc.n, dsc.r1 = c.shape
            df, sw = c.df, c.sw
            sp = _SparsePivot(df.nnz, df.fiber_of.data_ptr(), df.pivot_index.data_ptr(),
                              df.values.data_ptr(),
                              sw.t_map.data_ptr() if sw.t_map is not None else None,
                              sw.s_map.data_ptr() if sw.s_map is not None else None,
                              df.R, df.indptr.data_ptr())
        else:
            c = c.contiguous()
            keep.append(c)
            dsc.kind = 0
            dsc.r0, dsc.n, dsc.r1 = (int(x) for x in c.shape)
            dsc.data = c.data_ptr()
    kind = {"static": 0, "dynamic": 1, "fixed": 2}[policy.kind]
    targets = nat.i64_array(policy.targets) if kind == 2 else None
    outs = (nat.ctypes.c_void_p * d)()
    shapes = (nat.ctypes.c_int64 * (3 * d))()
    zero = nat.ctypes.c_int32(0)
    vp = nat.ctypes.c_void_p
    cast = nat.ctypes.cast
    nat.check(nat.lib().ftt_sweep_rounding(
        nat.context(), d, pivot, cast(descs, vp),
        cast(nat.ctypes.pointer(sp), vp) if sp is not None else None, kind,
        float(policy.delta), float(policy.left), float(policy.right),
        cast(targets, vp) if targets is not None else None, 1 if kind == 0 else 0,
        cast(outs, vp), cast(shapes, vp), nat.ctypes.byref(zero)), "ftt_sweep_rounding")
    if zero.value:
        return None
    return [torch.as_tensor(_NativeCore(outs[k], shapes[3 * k:3 * k + 3]), device="cuda")
            for k in range(d)]


def _sweep_rounding_python(cores, pivot: int, policy: _Trunc):
    """_sweep_rounding (fasttt.py:324-356) on device cores, one C-ABI call per
    step; 0/1 cores are SideCore objects whose contractions are scatters.
    Returns dense device cores, or None for the zero train."""
    torch = _torch()
    lib, ctx = nat.lib(), nat.context()
    cs = list(cores)
    d = len(cs)
    hint = None  # previous step's rank: sketch width of the low-rank path
    for k in range(pivot, d - 1):  # :334-341
        C = cs[k]
        r0, n, r1 = (int(x) for x in C.shape)
        m = r0 * n
        s = None
        if isinstance(C, SparsePivotCore):
            s, rest2 = _sparse_first_step(C, m, r1, policy.delta_first(k), hint,
                                          policy.kind == "static")
            if s is None:  # certificate rejected (or not applicable): dense operand
                C = cs[k] = C.dense()
                s, rest2 = dev_svd_values(C, m, r1, r1, True), 0.0
        if s is None:
            s, rest2 = dev_svd_truncate(C, m, r1, r1, True, policy.delta_first(k), hint,
                                        policy.kind == "static")
        rank, _ = policy.first(k, s, (m, r1), rest2)
        hint = rank
        if rank == 0:
            return None
        U, V = dev_svd_vectors(m, r1, rank, True, False, True)  # V: carry (r1 x rank) col-major
        cs[k] = U.reshape(r0, n, rank)
        nxt = cs[k + 1]
        if isinstance(nxt, SideCore):
            new = _empty((rank, nxt.n * nxt.r_other))
            nat.check(lib.ftt_scatter_cols(ctx, rank, nxt.K, nat.ptr(nxt.kept), nat.ptr(V), r1,
                                           nxt.n * nxt.r_other, nat.ptr(new)), "ftt_scatter_cols")
            cs[k + 1] = new.reshape(rank, nxt.n, nxt.r_other)
        else:
            a, nn, c = (int(x) for x in nxt.shape)
            new = _empty((rank, nn * c))
            dgemm(0, 0, nn * c, rank, r1, 1.0, nxt, nn * c, V, r1, 0.0, new, nn * c)
            cs[k + 1] = new.reshape(rank, nn, c)
    for k in range(d - 1, pivot, -1):  # :342-347
        C = cs[k] = _as_dense(cs[k]) if isinstance(cs[k], SparsePivotCore) else cs[k]
        r0, n, r1 = (int(x) for x in C.shape)
        Q, R = dev_qr(C, n * r1, r0, n * r1)
        q = int(Q.shape[0])
        cs[k] = Q.reshape(q, n, r1)
        P = cs[k - 1]
        if isinstance(P, SideCore):  # only when the QR sweep meets a 0/1 core
            P = P.dense()
        a, b, c = (int(x) for x in P.shape)
        Y = _empty((a * b, q))
        dgemm(0, 0, q, a * b, c, 1.0, R, q, P, c, 0.0, Y, q)
        cs[k - 1] = Y.reshape(a, b, q)
    for k in range(pivot, 0, -1):  # :348-355
        C = cs[k] = _as_dense(cs[k]) if isinstance(cs[k], SparsePivotCore) else cs[k]
        r0, n, r1 = (int(x) for x in C.shape)
        s, rest2 = dev_svd_truncate(C, n * r1, r0, n * r1, False, policy.delta_second(k), hint,
                                    policy.kind == "static")
        rank, _ = policy.second(k, s, (n * r1, r0), rest2)
        hint = rank
        if rank == 0:
            return None
        U, V = dev_svd_vectors(n * r1, r0, rank, False, True, True)  # V: carry (r0 x rank) row-major
        cs[k] = U.reshape(rank, n, r1)
        prv = cs[k - 1]
        if isinstance(prv, SideCore):
            new = _empty((prv.r_other * prv.n, rank))
            nat.check(lib.ftt_scatter_rows(ctx, prv.K, rank, nat.ptr(prv.kept), nat.ptr(V), rank,
                                           prv.r_other * prv.n, nat.ptr(new)), "ftt_scatter_rows")
            cs[k - 1] = new.reshape(prv.r_other, prv.n, rank)
        else:
            a, b, c = (int(x) for x in prv.shape)
            Y = _empty((a * b, rank))
            dgemm(0, 0, rank, a * b, c, 1.0, V, rank, prv, c, 0.0, Y, rank)
            cs[k - 1] = Y.reshape(a, b, rank)
    out = [_as_dense(c) for c in cs]
    del torch
    return out


def _sparse_first_step(spc: SparsePivotCore, m: int, n: int, delta, hint, interval_ok: bool):
    """dev_svd_truncate's low-rank branch on the entries of the pivot core;
    (None, 0) when it does not apply or its certificate is rejected."""
    if delta is None or not delta > 0.0:
        return None, 0.0
    k = lowrank_k(min(m, n), hint)
    if not k or k > 64:
        return None, 0.0
    s, rest2, acc = spc.svd_lowrank(k, delta)
    if acc == 2:
        return s, rest2
    if acc == 1 and interval_ok:
        shape = (m, n)
        if tail_rank(s, delta, shape, 0.0) == tail_rank(s, delta, shape, rest2):
            return s, rest2
    return None, 0.0


def _make_policy(budget: TruncationBudget, d: int, norm: float):
    pivot = budget.pivot
    denom = math.sqrt(pivot) + math.sqrt(d - 1 - pivot)
    if budget.mode == "static":
        if budget.delta_left is not None or budget.delta_right is not None:
            delta = budget.delta_left if budget.delta_left is not None else budget.delta_right
        else:
            delta = budget.eps * norm / denom if denom else 0.0
        return _Trunc("static", d, delta=delta)
    if budget.mode == "dynamic":
        right = budget.delta_right if budget.delta_right is not None else (
            math.sqrt(d - 1 - pivot) / denom * budget.eps * norm if denom else 0.0)
        left = budget.delta_left if budget.delta_left is not None else (
            math.sqrt(pivot) / denom * budget.eps * norm if denom else 0.0)
        return _Trunc("dynamic", d, left=left, right=right)
    return None


def _fixed_targets(budget: TruncationBudget, dims):
    d = len(dims)
    targets = budget.fixed_ranks
    if isinstance(targets, (int, np.integer)):
        targets = (int(targets),) * (d - 1)
    targets = full_ranks(dims, targets)
    if any(r < 1 for r in targets[1:-1]):
        raise ValueError("interior rank targets must be positive")
    return targets


def _check_pivot_orthogonal_device(cores_d, pivot: int, tol: float = 1e-8) -> None:
    """_check_pivot_orthogonal (fasttt.py:303-321): max|M^T M - I| per side core."""
    lib, ctx = nat.lib(), nat.context()
    for k in range(len(cores_d)):
        if k == pivot:
            continue
        r0, n, r1 = (int(x) for x in cores_d[k].shape)
        if k < pivot:  # columns of (r0 n x r1): G = M^T M (r1 x r1)
            G = _empty((r1, r1))
            dgemm(0, 1, r1, r1, r0 * n, 1.0, cores_d[k], r1, cores_d[k], r1, 0.0, G, r1)
            size = r1
        else:  # rows of (r0 x n r1): G = M M^T (r0 x r0)
            G = _empty((r0, r0))
            dgemm(1, 0, r0, r0, n * r1, 1.0, cores_d[k], n * r1, cores_d[k], n * r1, 0.0, G, r0)
            size = r0
        out = nat.ctypes.c_double(0.0)
        nat.check(lib.ftt_orth_defect(ctx, size, nat.ptr(G), size, nat.ctypes.byref(out)),
                  "ftt_orth_defect")
        if out.value > tol:
            side = "left" if k < pivot else "right"
            raise ContractViolationError(
                f"core {k} is not {side}-orthonormal; the train was not produced by "
                f"parallel_vector_round with pivot {pivot}")


def _round_dense_api(t: TTTensor, budget: TruncationBudget, mode: str) -> TTTensor:
    if budget.mode != mode:
        names = {"static": "static", "dynamic": "dynamic", "fixed_rank": "fixed-rank"}
        raise ValueError(f"{names[mode]} rounding got budget mode {budget.mode!r}")
    pivot = budget.pivot
    _check_pivot(pivot, t.ndim)
    cores_d = [to_device(c) for c in t.cores]
    _check_pivot_orthogonal_device(cores_d, pivot)
    d = t.ndim
    if d == 1:
        return TTTensor([c.copy() for c in t.cores])
    if mode == "fixed_rank":
        policy = _Trunc("fixed", d, targets=_fixed_targets(budget, t.dims))
    else:
        norm = math.sqrt(device_dot(cores_d[pivot].reshape(-1), None))
        policy = _make_policy(budget, d, norm)
    out = _sweep_rounding_device(cores_d, pivot, policy)
    if out is None:
        return tt_zero(t.dims)
    return TTTensor([c.cpu().numpy() for c in out], copy=False)


def efficient_tt_rounding(t: TTTensor, budget: TruncationBudget) -> TTTensor:
    """Static per-step tolerance eps*norm/(sqrt(p)+sqrt(d-1-p)) (fasttt.py:364-386)."""
    return _round_dense_api(t, budget, "static")


def dynamic_tt_rounding(t: TTTensor, budget: TruncationBudget) -> TTTensor:
    """Per-step tolerances that re-absorb unspent budget (fasttt.py:389-428)."""
    return _round_dense_api(t, budget, "dynamic")


def fixed_rank_rounding(t: TTTensor, budget: TruncationBudget) -> TTTensor:
    """Round to prescribed bond ranks (fasttt.py:431-453)."""
    return _round_dense_api(t, budget, "fixed_rank")


# ------------------------------------------------------------ error report
def _dev_tt_add_neg(a_cores, b_cores):
    """tt_add(a, tt_scale(b, -1)) on device cores (block-diagonal layout)."""
    torch = _torch()
    d = len(a_cores)
    if d == 1:
        return [a_cores[0] - b_cores[0]]
    out = []
    for k in range(d):
        ca, cb = a_cores[k], b_cores[k]
        if k == 0:
            out.append(torch.cat([ca, -cb], dim=2))
        elif k == d - 1:
            out.append(torch.cat([ca, cb], dim=0))
        else:
            ra0, n, ra1 = ca.shape
            rb0, _, rb1 = cb.shape
            c = torch.zeros((ra0 + rb0, n, ra1 + rb1), dtype=torch.float64, device="cuda")
            c[:ra0, :, :ra1] = ca
            c[ra0:, :, ra1:] = cb
            out.append(c)
    return out


def _dev_relative_error(ref_d, approx_d, norm):
    diff = _dev_tt_add_neg(ref_d, approx_d)
    ortho = dev_right_orthogonalize(diff)
    num = math.sqrt(device_dot(ortho[0].reshape(-1), None))
    if norm is None:
        norm = dev_tt_norm(ref_d)
    return num / norm if norm > 0 else (0.0 if num == 0.0 else math.inf)


def _diff_total(ref_shapes, approx_shapes):
    return sum((ra0 + rb0) * n * (ra1 + rb1)
               for (ra0, n, ra1), (rb0, _, rb1) in zip(ref_shapes, approx_shapes))


def tt_relative_error(reference: TTTensor, approx: TTTensor, norm: float | None = None) -> float:
    """``norm(reference - approx) / norm(reference)`` via the orthogonalised
    difference train (fasttt.py:561-584)."""
    if reference.dims != approx.dims:
        raise ValueError("trains must share mode extents")
    total = _diff_total([c.shape for c in reference.cores], [c.shape for c in approx.cores])
    if total > _ERROR_MEASURE_CAP:
        raise ValueError(f"difference train size {total} exceeds measurement cap")
    return _dev_relative_error([to_device(c) for c in reference.cores],
                               [to_device(c) for c in approx.cores], norm)


def _inner_error_device(coords_d, values_d, nnz, approx_d, na2=None):
    if na2 is None:
        na2 = device_dot(values_d, None)
    if na2 == 0.0:
        return 0.0 if dev_tt_norm(approx_d) == 0.0 else math.inf
    ent = dev_tt_entries(approx_d, coords_d)
    # <a, b> and |b|^2 with one host round trip (ftt_inner_terms)
    d = len(approx_d)
    cs = [c.contiguous() for c in approx_d]
    dims = [int(c.shape[1]) for c in cs]
    ranks = [int(cs[0].shape[0])] + [int(c.shape[2]) for c in cs]
    ptrs = (nat.ctypes.c_void_p * d)(*[c.data_ptr() for c in cs])
    terms = (nat.ctypes.c_double * 2)()
    nat.check(nat.lib().ftt_inner_terms(nat.context(), int(values_d.numel()), nat.ptr(values_d),
                                        nat.ptr(ent), d, nat.i64_array(dims), nat.i64_array(ranks),
                                        ptrs, terms), "ftt_inner_terms")
    dot, nb2 = float(terms[0]), max(float(terms[1]), 0.0)
    return math.sqrt(max(na2 - 2.0 * dot + nb2, 0.0) / na2)


def _inner_error_structured(df, sw: DeviceSweeps, approx_d, na2):
    """The inner-product identity with <a, b> evaluated on the fiber /
    sweep structure (ftt_inner_structured: one prefix vector per distinct
    prefix, one suffix vector per distinct suffix, a length-r_p dot per
    nonzero); None when the setup would cost more than the per-entry
    evaluation (very high ranks)."""
    d, p = len(approx_d), df.pivot
    cs = [c.contiguous() for c in approx_d]
    dims = [int(c.shape[1]) for c in cs]
    ranks = [1] + [int(c.shape[2]) for c in cs]
    steps = list(sw.left) + list(sw.right)
    counts = [int(k.shape[0]) for k, _ in steps]
    kl = counts[p - 1] if p > 0 else 1
    cost = sum(counts[k] * ranks[k] * ranks[k + 1] for k in range(p))
    cost += kl * dims[p] * ranks[p] * ranks[p + 1]
    cost += sum(counts[p + q] * ranks[d - 1 - q] * ranks[d - q] for q in range(d - 1 - p))
    if cost > 4e9 or na2 == 0.0:
        return None
    ptrs = (nat.ctypes.c_void_p * d)(*[c.data_ptr() for c in cs])
    kp = (nat.ctypes.c_void_p * max(len(steps), 1))(*[k.data_ptr() for k, _ in steps])
    dot = nat.ctypes.c_double(0.0)
    nat.check(nat.lib().ftt_inner_structured(
        nat.context(), d, nat.i64_array(dims), nat.i64_array(ranks), ptrs, p, kp,
        nat.i64_array(counts or [0]), df.R, nat.ptr(df.indptr), nat.ptr(df.pivot_index),
        nat.ptr(df.values), nat.ptr(sw.t_map), nat.ptr(sw.s_map), nat.ctypes.byref(dot)),
        "ftt_inner_structured")
    # the rounding sweeps leave cores 1..d-1 right-orthogonal, so the train's
    # norm is core 0's (same value as ftt_fasttt_lin's report terms)
    nb2 = math.sqrt(device_dot(cs[0].reshape(-1), None)) ** 2
    return math.sqrt(max(na2 - 2.0 * float(dot.value) + nb2, 0.0) / na2)


def sparse_inner_error(a: SparseTensor, approx: TTTensor) -> float:
    """Relative error via ``|a|^2 - 2<a,b> + |b|^2`` (fasttt.py:587-602)."""
    if a.shape != approx.dims:
        raise ValueError("tensor and train must share mode extents")
    approx_d = [to_device(c) for c in approx.cores]
    if a.nnz == 0:
        return 0.0 if dev_tt_norm(approx_d) == 0.0 else math.inf
    c, v = a.device_arrays()
    return _inner_error_device(c, v, a.nnz, approx_d)


@dataclass(frozen=True)
class DecompositionReport:
    """What a pipeline run did (fasttt.py:605-631)."""

    shape: tuple
    nnz: int
    pivot: int
    mode: str
    eps: float
    num_fibers: int
    ranks_lossless: tuple
    ranks: tuple
    eps_actual: float
    eps_actual_method: str
    eps_actual_inner: float | None
    flops_fasttt_model: float
    flops_ttsvd_model: float
    wall_time_s: float
    cpu_time_s: float
    warnings: tuple = ()


# ---------------------------------------------------------------- driver
class DeviceResult:
    """fasttt_device output: device cores + everything the report needs."""

    __slots__ = ("_cores", "slab", "shapes", "pivot", "mode", "eps", "num_fibers",
                 "ranks_lossless", "ranks", "eps_actual", "eps_actual_method", "eps_actual_inner",
                 "notes", "zero")

    def __init__(self, **kw):
        self._cores = kw.pop("cores", None)
        for k in self.__slots__[1:]:
            setattr(self, k, kw.get(k))

    @property
    def cores(self):
        """Device cores; a train the fused driver returned as one slab
        (``slab`` flat f64, ``shapes``) is split into views on first use."""
        if self._cores is None and self.slab is not None:
            out, off = [], 0
            for sh in self.shapes:
                n = sh[0] * sh[1] * sh[2]
                out.append(self.slab[off:off + n].view(sh))
                off += n
            self._cores = out
        return self._cores


def _normalize(eps, mode):
    if eps is None or eps == 0.0:
        eps = 1e-14
    if eps < 0:
        raise ValueError(f"eps must be nonnegative, got {eps}")
    if mode == "fixed":
        mode = "fixed_rank"
    if mode not in _MODES:
        raise ValueError(f"mode must be one of {_MODES}, got {mode!r}")
    return eps, mode


class _FastttResult(nat.ctypes.Structure):
    """ftt_fasttt_result (include/fasttt_b200.h)."""

    _fields_ = [("pivot", nat.ctypes.c_int32), ("zero", nat.ctypes.c_int32),
                ("fallback", nat.ctypes.c_int32), ("inner_valid", nat.ctypes.c_int32),
                ("lazy_pivot", nat.ctypes.c_int32), ("status_flags", nat.ctypes.c_int32),
                ("num_fibers", nat.ctypes.c_int64), ("step_counts", nat.ctypes.c_int64 * 32),
                ("kept_off", nat.ctypes.c_int64 * 32), ("pivot_shape", nat.ctypes.c_int64 * 3),
                ("out_shapes", nat.ctypes.c_int64 * 96), ("out_total", nat.ctypes.c_int64),
                ("na2", nat.ctypes.c_double), ("pnorm", nat.ctypes.c_double),
                ("dot", nat.ctypes.c_double), ("nb", nat.ctypes.c_double),
                ("fiber_slab", nat.ctypes.c_void_p), ("fixed_lin", nat.ctypes.c_void_p),
                ("indptr", nat.ctypes.c_void_p), ("fiber_of", nat.ctypes.c_void_p),
                ("pivot_index", nat.ctypes.c_void_p), ("values_f", nat.ctypes.c_void_p),
                ("kept_slab", nat.ctypes.c_void_p), ("maps_slab", nat.ctypes.c_void_p),
                ("out_slab", nat.ctypes.c_void_p), ("out_cores", nat.ctypes.c_void_p * 32)]


def _fused_structure(r: "_FastttResult", dims, nnz: int):
    """DeviceFibers / DeviceSweeps views over the buffers ftt_fasttt_lin
    returned (each slab is owned by one holder the views keep alive)."""
    from .coo import DeviceFibers

    torch = _torch()
    d, p, R = len(dims), int(r.pivot), int(r.num_fibers)
    fib = torch.as_tensor(_NativeCore(r.fiber_slab, (5 * nnz + 1,), "<i8"), device="cuda")
    df = DeviceFibers(tuple(dims), p, R, nnz, fib[:R], fib[nnz:nnz + R + 1],
                      fib[2 * nnz + 1:3 * nnz + 1], fib[3 * nnz + 1:4 * nnz + 1],
                      fib[4 * nnz + 1:5 * nnz + 1].view(torch.float64))
    nsteps = d - 1
    cnt = [int(r.step_counts[s]) for s in range(nsteps)]
    off = [int(r.kept_off[s]) for s in range(nsteps)]
    ktot = off[-1] + max(cnt[-1], 1) if nsteps else 1
    kb = torch.as_tensor(_NativeCore(r.kept_slab, (max(ktot, 1),), "<i8"), device="cuda")
    mb = torch.as_tensor(_NativeCore(r.maps_slab, (max(R, 1) * nsteps,), "<i8"), device="cuda")
    left, right = [], []
    t_map, r_prev, s_map, r_next = None, 1, None, 1
    for s in range(nsteps):
        kept = kb[off[s]:off[s] + cnt[s]]
        m = mb[s * max(R, 1):s * max(R, 1) + R]
        if s < p:
            left.append((kept, r_prev))
            t_map, r_prev = m, cnt[s]
        else:
            right.append((kept, r_next))
            s_map, r_next = m, cnt[s]
    return df, DeviceSweeps(left, t_map, r_prev, right, s_map, r_next)


def _fasttt_fused(a: SparseTensor, values_d, eps, pivot, mode, c_svd, report, values_ready):
    """fasttt_device through ftt_fasttt_lin (static / dynamic budgets): one
    native call from select_p to the report's inner-product terms; None when
    the native side asks for the step-by-step path."""
    torch = _torch()
    d, dims, nnz = a.ndim, a.shape, a.nnz
    lib, ctx = nat.lib(), nat.context()
    r = _FastttResult()
    ev = nat.ctypes.c_void_p(values_ready.cuda_event) if values_ready is not None else None
    chunks = a.take_lin_chunks()
    if chunks is not None:  # lin still arriving: the native side waits chunk by chunk
        ends, evs = chunks
        nat.check(lib.ftt_set_lin_chunks(
            ctx, len(ends), nat.i64_array(ends),
            (nat.ctypes.c_void_p * len(evs))(*[e.cuda_event for e in evs])), "ftt_set_lin_chunks")
    try:
        nat.check(lib.ftt_fasttt_lin(ctx, nat.ptr(a.device_lin()), nat.ptr(values_d), nnz, d,
                                     nat.i64_array(dims), -1 if pivot is None else int(pivot),
                                     0 if mode == "static" else 1, float(eps), float(c_svd),
                                     1 if report else 0, ev, nat.ctypes.byref(r)),
                  "ftt_fasttt_lin")
    except MemoryError as e:
        if "pivot core" in str(e):
            shape = tuple(int(x) for x in r.pivot_shape)
            raise MemoryError(f"pivot core {shape} does not fit in device memory") from e
        raise
    if r.fallback:
        return None
    if r.status_flags & 1:
        raise ValueError("matrix entries must be finite")
    free = lib.ftt_free_device
    vp = nat.ctypes.c_void_p
    notes = []
    zero = bool(r.zero)
    shapes = [tuple(int(x) for x in r.out_shapes[3 * k:3 * k + 3]) for k in range(d)]
    if r.out_slab:
        slab = torch.as_tensor(_NativeCore(r.out_slab, (max(int(r.out_total), 1),)), device="cuda")
        cores = None
    else:
        slab = None
        cores = [torch.as_tensor(_NativeCore(r.out_cores[k], shapes[k]), device="cuda")
                 for k in range(d)]
    p = int(r.pivot)
    cnt = [int(r.step_counts[s]) for s in range(d - 1)]
    bonds = [0] * (d - 1)
    for s in range(d - 1):
        bonds[s if s < p else d - 2 - (s - p)] = cnt[s]
    res = DeviceResult(cores=cores, slab=slab, shapes=shapes, pivot=p, mode=mode, eps=eps,
                       num_fibers=int(r.num_fibers), ranks_lossless=tuple(bonds),
                       ranks=tuple(sh[2] for sh in shapes[:-1]), notes=notes, zero=zero)
    structure = None
    if report:
        na2 = float(r.na2)
        if r.inner_valid:
            nb2 = float(r.nb) ** 2
            inner = math.sqrt(max(na2 - 2.0 * float(r.dot) + nb2, 0.0) / na2)
        else:
            coords_d, _ = a.device_arrays()
            inner = _inner_error_device(coords_d, values_d, nnz, res.cores, na2)
        # shapes of the lossless train (0/1 cores + pivot core)
        exact, rp, rn = [None] * d, 1, 1
        for s in range(d - 1):
            if s < p:
                exact[s] = (rp, dims[s], cnt[s])
                rp = cnt[s]
            else:
                k = d - 1 - (s - p)
                exact[k] = (cnt[s], dims[k], rn)
                rn = cnt[s]
        exact[p] = (rp, dims[p], rn)
        total = _diff_total(exact, shapes)
        if total <= _ERROR_MEASURE_CAP:
            df, sw = structure = _fused_structure(r, dims, nnz)
            train, _ = _structured_train(df, sw)
            res.eps_actual = _dev_relative_error([_as_dense(c) for c in train], res.cores,
                                                 math.sqrt(na2))
            res.eps_actual_method = "tt_difference"
        else:
            res.eps_actual = inner
            res.eps_actual_method = "inner_identity"
            notes.append("exact-difference error measure too large; reported value is the "
                         "inner-product identity (resolution ~1e-8)")
        res.eps_actual_inner = inner
    if structure is None:
        for ptr in (r.fiber_slab, r.kept_slab, r.maps_slab):
            if ptr:
                free(ctx, vp(ptr))
    return res


def fasttt_device(a: SparseTensor, coords_d, values_d, eps, pivot, mode, fixed_ranks,
                  precise_pivot, c_svd, report=True, values_ready=None) -> DeviceResult:
    """The decomposition on device arrays (COO already in HBM)."""
    d = a.ndim
    dims = a.shape
    nnz = a.nnz
    notes = []
    if (mode in ("static", "dynamic") and not precise_pivot and nnz and d >= 2
            and not _STEPWISE and __import__("os").environ.get("FTT_PY_SWEEP") != "1"):
        if pivot is not None:
            _check_pivot(pivot, d)
        res = _fasttt_fused(a, values_d, eps, pivot, mode, c_svd, report, values_ready)
        if res is not None:
            return res
    a._lin_arrived()  # (a chunked upload the fused call did not take over)
    if pivot is None:
        pivot = select_p(a, target_ranks=fixed_ranks if mode == "fixed_rank" else None,
                         precise=precise_pivot, c_svd=c_svd)
    _check_pivot(pivot, d)
    if nnz == 0:
        notes.append("input has no nonzeros; returning the zero train")
        return DeviceResult(cores=None, pivot=pivot, mode=mode, eps=eps, num_fibers=0,
                            ranks_lossless=(0,) * (d - 1), ranks=(1,) * (d - 1), eps_actual=0.0,
                            eps_actual_method="exact", eps_actual_inner=0.0, notes=notes, zero=True)
    lib, ctx = nat.lib(), nat.context()
    # the narrow QR steps report non-finite inputs through a device flag read
    # once at the end (the COO values are validated finite up front)
    nat.check(lib.ftt_set_deferred_checks(ctx, 1), "ftt_set_deferred_checks")
    try:
        if values_ready is not None:  # the values' H2D overlapped select_p
            _torch().cuda.current_stream().wait_event(values_ready)
        res = _fasttt_device_body(a, coords_d, values_d, eps, pivot, mode, fixed_ranks, notes,
                                  report)
    finally:
        nat.check(lib.ftt_set_deferred_checks(ctx, 0), "ftt_set_deferred_checks")
    flags = nat.ctypes.c_int32(0)
    nat.check(lib.ftt_take_status(ctx, nat.ctypes.byref(flags)), "ftt_take_status")
    if flags.value & 1:
        raise ValueError("matrix entries must be finite")
    return res


def _fasttt_device_body(a, coords_d, values_d, eps, pivot, mode, fixed_ranks, notes, report):
    d = a.ndim
    dims = a.shape
    nnz = a.nnz
    df = fibers_device(dims, pivot, coords_d, values_d, nnz, lin_d=a.device_lin())
    if d == 1:
        # the reference's FiberSet rejects its own d = 1 output (tensor.py:326-329)
        raise ValueError("inconsistent fiber index pointers")
    sw = index_sweeps_device(df)
    ranks_lossless = _lossless_ranks_from(sw, d)
    na2 = device_dot(values_d, None) if report else None
    cores, pnorm = _structured_train(df, sw, lazy_pivot=mode != "fixed_rank", na2=na2)
    budget = TruncationBudget(eps=eps, pivot=pivot, mode=mode, fixed_ranks=fixed_ranks)
    if mode == "fixed_rank":
        policy = _Trunc("fixed", d, targets=_fixed_targets(budget, dims))
    else:
        policy = _make_policy(budget, d, pnorm)
    out = _sweep_rounding_device(cores, pivot, policy)
    zero = out is None
    if zero:
        torch = _torch()
        out = [torch.zeros((1, n, 1), dtype=torch.float64, device="cuda") for n in dims]
    ranks = tuple(int(c.shape[2]) for c in out[:-1])
    res = DeviceResult(cores=out, pivot=pivot, mode=mode, eps=eps, num_fibers=df.R,
                       ranks_lossless=ranks_lossless, ranks=ranks, notes=notes, zero=zero)
    if report:
        if na2 is None:
            na2 = device_dot(values_d, None)
        norm_a = math.sqrt(na2)
        inner = _inner_error_structured(df, sw, out, na2)
        if inner is None:
            if coords_d is None:
                coords_d, _ = a.device_arrays()
            inner = _inner_error_device(coords_d, values_d, nnz, out, na2)
        exact_shapes = [tuple(c.shape) for c in cores]
        total = _diff_total(exact_shapes, [tuple(c.shape) for c in out])
        if total <= _ERROR_MEASURE_CAP:
            exact_d = [_as_dense(c) for c in cores]
            res.eps_actual = _dev_relative_error(exact_d, out, norm_a)
            res.eps_actual_method = "tt_difference"
        else:
            res.eps_actual = inner
            res.eps_actual_method = "inner_identity"
            notes.append("exact-difference error measure too large; reported value is the "
                         "inner-product identity (resolution ~1e-8)")
        res.eps_actual_inner = inner
    return res


_STAGE_MAX = 256 << 20  # cores up to this size go through the reused staging buffer
_stage = __import__("threading").local()


def _slab_to_host(slab, shapes):
    """D2H of a train held as one device slab: one copy into the reused
    pinned staging buffer, one sync, numpy views of one host array."""
    torch = _torch()
    total = int(slab.numel())
    buf = getattr(_stage, "buf", None)
    if buf is None or buf.numel() < total:
        buf = torch.empty(max(total, 1 << 16), dtype=torch.float64, pin_memory=True)
        _stage.buf = buf
    buf[:total].copy_(slab, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    flat = buf.numpy()[:total].copy()
    out, off = [], 0
    for sh in shapes:
        n = sh[0] * sh[1] * sh[2]
        out.append(flat[off:off + n].reshape(sh))
        off += n
    return out


def _cores_to_host(cores):
    """D2H of the final cores with one stream sync.  Up to _STAGE_MAX bytes
    they land in a per-thread pinned staging buffer that is reused across
    calls and are copied out into ordinary numpy arrays (a caller holding the
    previous result no longer forces torch's host allocator to pin a fresh
    block inside the call: that showed up as 15-45 ms outliers on config 5);
    larger trains land in fresh pinned buffers (``.cpu()`` into pageable
    memory: 0.9 s instead of 34 ms for config 3's 1.9 GB of cores)."""
    torch = _torch()
    sizes = [int(c.numel()) for c in cores]
    total = sum(sizes)
    if 8 * total > _STAGE_MAX:
        host = [torch.empty(tuple(c.shape), dtype=c.dtype, pin_memory=True) for c in cores]
        for h, c in zip(host, cores):
            h.copy_(c, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return [h.numpy() for h in host]
    buf = getattr(_stage, "buf", None)
    if buf is None or buf.numel() < total:
        buf = torch.empty(max(total, 1 << 16), dtype=torch.float64, pin_memory=True)
        _stage.buf = buf
    off = 0
    for n, c in zip(sizes, cores):
        buf[off:off + n].copy_(c.reshape(-1), non_blocking=True)
        off += n
    torch.cuda.current_stream().synchronize()
    flat = buf.numpy()[:total].copy()
    out, off = [], 0
    for n, c in zip(sizes, cores):
        out.append(flat[off:off + n].reshape(tuple(c.shape)))
        off += n
    return out


def fasttt(a: SparseTensor, eps: float | None = 1e-14, pivot: int | None = None,
           mode: str = "static", fixed_ranks=None, precise_pivot: bool = False,
           c_svd: float = 1.0):
    """Convert a sparse tensor to train format and round it
    (fasttt.py:634-749). Returns ``(TTTensor, DecompositionReport)``."""
    if not isinstance(a, SparseTensor):
        raise TypeError("fasttt expects a SparseTensor")
    wall0 = time.perf_counter()
    cpu0 = time.process_time()
    eps, mode = _normalize(eps, mode)
    ready = None
    if a.nnz:
        # lin + values only (no coordinate rows); the values' copy runs on a
        # side stream under select_p's counts
        # (a large lin arrives in chunks: the fused call starts on the first)
        _, values_d, ready = a.device_lin_values(keep_chunks=True)
    else:
        values_d = None
    res = fasttt_device(a, None, values_d, eps, pivot, mode, fixed_ranks, precise_pivot, c_svd,
                        values_ready=ready)
    if res.zero and res.cores is None:
        tt = tt_zero(a.shape)
        return tt, DecompositionReport(
            shape=a.shape, nnz=0, pivot=res.pivot, mode=mode, eps=eps, num_fibers=0,
            ranks_lossless=res.ranks_lossless, ranks=tt.ranks[1:-1], eps_actual=0.0,
            eps_actual_method="exact", eps_actual_inner=0.0, flops_fasttt_model=0.0,
            flops_ttsvd_model=0.0, wall_time_s=time.perf_counter() - wall0,
            cpu_time_s=time.process_time() - cpu0, warnings=tuple(res.notes))
    if res.slab is not None and res._cores is None:
        tt = TTTensor(_slab_to_host(res.slab, res.shapes), copy=False)
    else:
        tt = TTTensor(_cores_to_host(res.cores), copy=False)
    report = DecompositionReport(
        shape=a.shape, nnz=a.nnz, pivot=res.pivot, mode=mode, eps=eps, num_fibers=res.num_fibers,
        ranks_lossless=res.ranks_lossless, ranks=tt.ranks[1:-1], eps_actual=res.eps_actual,
        eps_actual_method=res.eps_actual_method, eps_actual_inner=res.eps_actual_inner,
        flops_fasttt_model=flops_fasttt(a.shape, res.pivot, res.ranks_lossless, tt.ranks, c_svd),
        flops_ttsvd_model=flops_ttsvd(a.shape, tt.ranks, c_svd),
        wall_time_s=time.perf_counter() - wall0, cpu_time_s=time.process_time() - cpu0,
        warnings=tuple(res.notes))
    return tt, report
