"""Tensor trains: host value types of the drop-in API plus their device-side
algebra (reference ttformat.py names on the FastTT path).

``TTTensor`` / ``TTMatrix`` / ``QuasiPermMatrix`` / ``StructuredTT`` are the
immutable host containers the reference API returns (ttformat.py:55-101,
219-365, 454-504). The train algebra used by the decomposition and its report
-- ``tt_entries``, ``tt_norm``, ``tt_right_orthogonalize`` -- runs on the GPU
(ftt_tt_entries, ftt_dgemm, ftt_qr_f64). ``tt_add`` / ``tt_scale`` /
``tt_split_mpo`` are pure data layout.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as nat
from .coo import (
    FiberSet,
    FormatError,
    SparseTensor,
    check_shape,
    delinearize,
)

__all__ = [
    "TTTensor",
    "TTMatrix",
    "QuasiPermMatrix",
    "StructuredTT",
    "tt_zero",
    "tt_entries",
    "tt_norm",
    "tt_scale",
    "tt_add",
    "tt_right_orthogonalize",
    "tensorize_matrix",
    "tt_split_mpo",
]


class TTTensor:
    """Train with 3-way cores ``(r_{k-1}, n_k, r_k)`` and unit edge ranks."""

    __slots__ = ("cores",)

    def __init__(self, cores, copy: bool = True):
        cs = [np.asarray(c, dtype=np.float64) for c in cores]
        if not cs:
            raise ValueError("a train needs at least one core")
        for k, c in enumerate(cs):
            if c.ndim != 3:
                raise ValueError(f"core {k} must be 3-way, got shape {c.shape}")
        if cs[0].shape[0] != 1 or cs[-1].shape[2] != 1:
            raise ValueError("edge ranks must be 1")
        for k in range(len(cs) - 1):
            if cs[k].shape[2] != cs[k + 1].shape[0]:
                raise ValueError(
                    f"bond mismatch between cores {k} and {k + 1}: "
                    f"{cs[k].shape[2]} vs {cs[k + 1].shape[0]}")
        if copy:
            cs = [np.ascontiguousarray(c) for c in cs]
            for c in cs:
                c.setflags(write=False)
        object.__setattr__(self, "cores", tuple(cs))

    def __setattr__(self, name, value):
        raise AttributeError("TTTensor is immutable")

    @property
    def ndim(self) -> int:
        return len(self.cores)

    @property
    def dims(self) -> tuple[int, ...]:
        return tuple(int(c.shape[1]) for c in self.cores)

    @property
    def ranks(self) -> tuple[int, ...]:
        return (1,) + tuple(int(c.shape[2]) for c in self.cores)

    @property
    def num_params(self) -> int:
        return int(sum(c.size for c in self.cores))

    def __repr__(self) -> str:
        return f"TTTensor(dims={self.dims}, ranks={self.ranks})"


def tt_zero(dims) -> TTTensor:
    """All-zero train of rank 1 (ttformat.py:104-107)."""
    return TTTensor([np.zeros((1, n, 1)) for n in check_shape(dims)])


class QuasiPermMatrix:
    """0/1 matrix with exactly one 1 per column, stored as column -> row."""

    __slots__ = ("n_rows", "n_cols", "col_to_row")

    def __init__(self, n_rows: int, n_cols: int, col_to_row):
        n_rows, n_cols = int(n_rows), int(n_cols)
        m = np.ascontiguousarray(col_to_row, dtype=np.int64)
        if n_rows < 0 or n_cols < 0:
            raise ValueError("matrix extents must be nonnegative")
        if m.shape != (n_cols,):
            raise ValueError(f"col_to_row must have shape ({n_cols},)")
        if n_cols and (m.min() < 0 or m.max() >= n_rows):
            raise ValueError("column map points outside the row range")
        m.setflags(write=False)
        object.__setattr__(self, "n_rows", n_rows)
        object.__setattr__(self, "n_cols", n_cols)
        object.__setattr__(self, "col_to_row", m)

    def __setattr__(self, name, value):
        raise AttributeError("QuasiPermMatrix is immutable")

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols))
        out[self.col_to_row, np.arange(self.n_cols)] = 1.0
        return out

    def __repr__(self) -> str:
        return f"QuasiPermMatrix(shape={self.shape})"


class StructuredTT:
    """Exact train of a sparse tensor in index form (ttformat.py:281-365):
    every interior bond is the fiber count R, non-pivot cores are 0/1 maps."""

    __slots__ = ("fibers",)

    def __init__(self, fibers: FiberSet):
        if not isinstance(fibers, FiberSet):
            raise TypeError("StructuredTT is built from a FiberSet")
        object.__setattr__(self, "fibers", fibers)

    def __setattr__(self, name, value):
        raise AttributeError("StructuredTT is immutable")

    @property
    def shape(self):
        return self.fibers.shape

    @property
    def pivot(self) -> int:
        return self.fibers.pivot

    @property
    def num_fibers(self) -> int:
        return self.fibers.num_fibers

    @property
    def ndim(self) -> int:
        return len(self.shape)

    @property
    def ranks(self):
        return (1,) + (self.num_fibers,) * (self.ndim - 1) + (1,)

    def mode_index(self, k: int) -> np.ndarray:
        if k == self.pivot or not 0 <= k < self.ndim:
            raise ValueError(f"mode {k} is the pivot or out of range")
        return self.fibers.fixed_coords[:, k if k < self.pivot else k - 1]

    def perm_core(self, k: int) -> QuasiPermMatrix:
        r = self.num_fibers
        n = self.shape[k]
        ik = self.mode_index(k)
        ids = np.arange(r, dtype=np.int64)
        if k < self.pivot:
            prev = ids if k > 0 else np.zeros(r, np.int64)
            return QuasiPermMatrix((r if k > 0 else 1) * n, r, prev * n + ik)
        last = k == self.ndim - 1
        nxt = np.zeros(r, np.int64) if last else ids
        rn = 1 if last else r
        return QuasiPermMatrix(n * rn, r, ik * rn + nxt)

    def __repr__(self) -> str:
        return f"StructuredTT(shape={self.shape}, pivot={self.pivot}, fibers={self.num_fibers})"


class TTMatrix:
    """Operator train with 4-way cores ``(r_{k-1}, m_k, n_k, r_k)``."""

    __slots__ = ("cores",)

    def __init__(self, cores, copy: bool = True):
        cs = [np.asarray(c, dtype=np.float64) for c in cores]
        if not cs:
            raise ValueError("an operator train needs at least one core")
        for k, c in enumerate(cs):
            if c.ndim != 4:
                raise ValueError(f"core {k} must be 4-way, got shape {c.shape}")
        if cs[0].shape[0] != 1 or cs[-1].shape[3] != 1:
            raise ValueError("edge ranks must be 1")
        for k in range(len(cs) - 1):
            if cs[k].shape[3] != cs[k + 1].shape[0]:
                raise ValueError(f"bond mismatch between cores {k} and {k + 1}")
        if copy:
            cs = [np.ascontiguousarray(c) for c in cs]
            for c in cs:
                c.setflags(write=False)
        object.__setattr__(self, "cores", tuple(cs))

    def __setattr__(self, name, value):
        raise AttributeError("TTMatrix is immutable")

    @property
    def ndim(self) -> int:
        return len(self.cores)

    @property
    def row_dims(self):
        return tuple(int(c.shape[1]) for c in self.cores)

    @property
    def col_dims(self):
        return tuple(int(c.shape[2]) for c in self.cores)

    @property
    def ranks(self):
        return (1,) + tuple(int(c.shape[3]) for c in self.cores)

    @property
    def num_params(self) -> int:
        return int(sum(c.size for c in self.cores))

    def __repr__(self) -> str:
        return f"TTMatrix(row_dims={self.row_dims}, col_dims={self.col_dims}, ranks={self.ranks})"


def _factor_dims(dims, total, what):
    dims = check_shape(dims)
    if math.prod(dims) != total:
        raise ValueError(f"{what} {dims} do not factor the matrix extent {total}")
    return dims


def tensorize_matrix(m, row_dims, col_dims, device: bool = False) -> SparseTensor:
    """Matrix -> fused ``d``-way tensor, ``f_i = x_i * col_dims[i] + y_i``
    (ttformat.py:414-433). Duplicates are coalesced first (scipy COO).

    ``device=True`` does the fusing, the canonical sort and the duplicate
    coalescing on the GPU (``ftt_tensorize_matrix``): only the matrix
    entries (24 B each) cross PCIe and the fused COO stays resident for the
    decomposition."""
    import scipy.sparse

    if not scipy.sparse.issparse(m):
        m = scipy.sparse.coo_matrix(np.asarray(m, dtype=np.float64))
    rdims = _factor_dims(row_dims, m.shape[0], "row factors")
    cdims = _factor_dims(col_dims, m.shape[1], "column factors")
    if len(rdims) != len(cdims):
        raise ValueError("row and column factorizations need equal length")
    if device:
        return _tensorize_device(m.tocoo(), rdims, cdims)
    m = m.tocsr().tocoo()
    x = delinearize(rdims, m.row.astype(np.int64))
    y = delinearize(cdims, m.col.astype(np.int64))
    fused = x * np.asarray(cdims, dtype=np.int64) + y
    return SparseTensor(tuple(a * b for a, b in zip(rdims, cdims)), fused, m.data)


def _tensorize_device(m, rdims, cdims) -> SparseTensor:
    torch = nat.torch_mod()
    vals = np.asarray(m.data, dtype=np.float64)
    if not np.isfinite(vals).all():
        raise FormatError("tensor values must be finite")
    d = len(rdims)
    dims = tuple(a * b for a, b in zip(rdims, cdims))
    nnz = int(vals.shape[0])
    rows = to_device(np.asarray(m.row, dtype=np.int64))
    cols = to_device(np.asarray(m.col, dtype=np.int64))
    vd = to_device(vals)
    coords = torch.empty((max(nnz, 1), d), dtype=torch.int64, device="cuda")
    vout = torch.empty(max(nnz, 1), dtype=torch.float64, device="cuda")
    kept = nat.ctypes.c_int64(0)
    nat.check(nat.lib().ftt_tensorize_matrix(nat.context(), nnz, nat.ptr(rows), nat.ptr(cols),
                                             nat.ptr(vd), d, nat.i64_array(rdims),
                                             nat.i64_array(cdims), nat.ptr(coords), nat.ptr(vout),
                                             nat.ctypes.byref(kept)), "ftt_tensorize_matrix")
    k = int(kept.value)
    return SparseTensor._from_canonical_device(dims, coords[:k].contiguous(), vout[:k].contiguous())


def tt_split_mpo(t: TTTensor, row_dims, col_dims) -> TTMatrix:
    """Fused train -> operator train: a reshape of every core (ttformat.py:507-518)."""
    rdims, cdims = check_shape(row_dims), check_shape(col_dims)
    fused = tuple(a * b for a, b in zip(rdims, cdims))
    if t.dims != fused:
        raise ValueError(f"train dims {t.dims} do not match fused dims {fused}")
    return TTMatrix([c.reshape(c.shape[0], a, b, c.shape[2])
                     for c, a, b in zip(t.cores, rdims, cdims)])


def tt_scale(t: TTTensor, alpha: float) -> TTTensor:
    cs = list(t.cores)
    cs[0] = cs[0] * float(alpha)
    return TTTensor(cs)


def _block_diag_cores(a_shapes_cores, b_cores):
    """tt_add layout (ttformat.py:157-182) for numpy or torch cores."""
    d = len(a_shapes_cores)
    out = []
    for k in range(d):
        ca, cb = a_shapes_cores[k], b_cores[k]
        if d == 1:
            out.append(ca + cb)
            continue
        if k == 0:
            out.append(_cat(ca, cb, 2))
        elif k == d - 1:
            out.append(_cat(ca, cb, 0))
        else:
            ra0, n, ra1 = ca.shape
            rb0, _, rb1 = cb.shape
            c = _zeros_like(ca, (ra0 + rb0, n, ra1 + rb1))
            c[:ra0, :, :ra1] = ca
            c[ra0:, :, ra1:] = cb
            out.append(c)
    return out


def _cat(a, b, axis):
    if isinstance(a, np.ndarray):
        return np.concatenate([a, b], axis=axis)
    return nat.torch_mod().cat([a, b], dim=axis)


def _zeros_like(a, shape):
    if isinstance(a, np.ndarray):
        return np.zeros(shape)
    return nat.torch_mod().zeros(shape, dtype=a.dtype, device=a.device)


def tt_add(a: TTTensor, b: TTTensor) -> TTTensor:
    if a.dims != b.dims:
        raise ValueError(f"dims differ: {a.dims} vs {b.dims}")
    return TTTensor(_block_diag_cores(list(a.cores), list(b.cores)))


# ----------------------------------------------------------------- device
def to_device(arr):
    torch = nat.torch_mod()
    return torch.from_numpy(np.ascontiguousarray(arr)).to("cuda")


def dgemm(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc):
    nat.check(nat.lib().ftt_dgemm(nat.context(), int(ta), int(tb), int(m), int(n), int(k),
                                  float(alpha), nat.ptr(A), int(lda), nat.ptr(B), int(ldb),
                                  float(beta), nat.ptr(C), int(ldc)), "ftt_dgemm")


def dev_qr(A, m, n, lda):
    """Column-major m x n at A -> (Q col-major m x k as torch (k, m),
    R col-major k x n as torch (n, k)); diag(R) >= 0 (linalg.py:128-140)."""
    torch = nat.torch_mod()
    k = min(m, n)
    Q = torch.empty((k, m), dtype=torch.float64, device="cuda")
    R = torch.empty((n, k), dtype=torch.float64, device="cuda")
    if k:
        nat.check(nat.lib().ftt_qr_f64(nat.context(), int(m), int(n), nat.ptr(A), int(lda),
                                       nat.ptr(Q), int(m), nat.ptr(R), int(k)), "ftt_qr_f64")
    return Q, R


def dev_tt_entries(cores_d, coords_d):
    """Entries of the device train at the (n, d) int64 device coordinates."""
    torch = nat.torch_mod()
    d = len(cores_d)
    n = int(coords_d.shape[0])
    out = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    if n == 0:
        return out[:0]
    dims = [int(c.shape[1]) for c in cores_d]
    ranks = [1] + [int(c.shape[2]) for c in cores_d]
    ptrs = (nat.ctypes.c_void_p * d)(*[c.data_ptr() for c in cores_d])
    nat.check(nat.lib().ftt_tt_entries(nat.context(), d, nat.i64_array(dims), nat.i64_array(ranks),
                                       ptrs, nat.ptr(coords_d), n, nat.ptr(out)), "ftt_tt_entries")
    return out[:n]


def dev_tt_norm(cores_d) -> float:
    """Train Frobenius norm by contracting it with itself (ttformat.py:198-203):
    ftt_tt_norm, two DMMA GEMMs per core and one host round trip."""
    d = len(cores_d)
    dims = [int(c.shape[1]) for c in cores_d]
    ranks = [int(cores_d[0].shape[0])] + [int(c.shape[2]) for c in cores_d]
    cs = [c.contiguous() for c in cores_d]
    ptrs = (nat.ctypes.c_void_p * d)(*[c.data_ptr() for c in cs])
    out = nat.ctypes.c_double(0.0)
    nat.check(nat.lib().ftt_tt_norm(nat.context(), d, nat.i64_array(dims), nat.i64_array(ranks),
                                    ptrs, nat.ctypes.byref(out)), "ftt_tt_norm")
    return float(out.value)


def dev_right_orthogonalize(cores_d):
    """QR sweep right to left (ttformat.py:206-216) on device cores."""
    torch = nat.torch_mod()
    cs = list(cores_d)
    for k in range(len(cs) - 1, 0, -1):
        r0, n, r1 = (int(x) for x in cs[k].shape)
        Q, R = dev_qr(cs[k], n * r1, r0, n * r1)
        q = Q.shape[0]
        cs[k] = Q.reshape(q, n, r1)
        a, b, c = (int(x) for x in cs[k - 1].shape)
        Y = torch.empty((a * b, q), dtype=torch.float64, device="cuda")
        dgemm(0, 0, q, a * b, c, 1.0, R, q, cs[k - 1], c, 0.0, Y, q)
        cs[k - 1] = Y.reshape(a, b, q)
    return cs


def _checked_indices(coords, dims, batch):
    """numpy's indexing contract of the reference's per-batch core slicing
    (ttformat.py:124-136): an index outside [-n, n) raises IndexError --
    the first batch holding one, its lowest such mode, that mode's first
    offending value -- and negative indices wrap.  The device kernels then
    only ever see indices in [0, n)."""
    lim = np.asarray(dims, dtype=np.int64)
    bad = (coords >= lim) | (coords < -lim)
    if bad.any():
        row = int(np.argmax(bad.any(axis=1)))
        lo = row - row % max(int(batch), 1)
        blk = bad[lo:lo + batch]
        k = int(np.argmax(blk.any(axis=0)))
        v = int(coords[lo + int(np.argmax(blk[:, k])), k])
        raise IndexError(f"index {v} is out of bounds for axis 1 with size {dims[k]}")
    if (coords < 0).any():
        coords = np.where(coords < 0, coords + lim, coords)
    return coords


def tt_entries(t: TTTensor, coords, batch: int = 1024) -> np.ndarray:
    """Entries at ``(n, d)`` coordinates (ttformat.py:124-136), on the GPU."""
    coords = np.asarray(coords, dtype=np.int64)
    if coords.ndim != 2 or coords.shape[1] != t.ndim:
        raise ValueError(f"coords must be (n, {t.ndim})")
    if coords.shape[0] == 0:
        return np.zeros(0)
    coords = _checked_indices(coords, t.dims, batch)
    cores_d = [to_device(c) for c in t.cores]
    return dev_tt_entries(cores_d, to_device(coords)).cpu().numpy()


def tt_norm(t: TTTensor) -> float:
    return dev_tt_norm([to_device(c) for c in t.cores])


def tt_right_orthogonalize(t: TTTensor) -> TTTensor:
    cs = dev_right_orthogonalize([to_device(c) for c in t.cores])
    return TTTensor([c.cpu().numpy() for c in cs], copy=False)
