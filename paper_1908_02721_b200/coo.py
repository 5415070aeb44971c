"""COO sparse tensors, fibers and C-order index arithmetic (drop-in for the
reference's ``tensor.py`` / ``errors.py`` names on the FastTT path).

``SparseTensor`` and ``FiberSet`` are the input/output *containers* of the
reference API: validated, canonical, immutable host arrays, exactly as the
reference defines them (tensor.py:103-197, 305-371). Everything computed from
them on the decomposition path -- fiber extraction, norms -- runs on the GPU
(``extract_nonzero_fibers`` -> ``ftt_extract_fibers``; ``frobenius_norm`` ->
``ftt_dot``).
"""

from __future__ import annotations

import math
import operator

import numpy as np

from . import _native as nat

__all__ = [
    "FormatError",
    "ContractViolationError",
    "DENSE_CAP",
    "SparseTensor",
    "FiberSet",
    "check_shape",
    "size_of",
    "linearize",
    "delinearize",
    "frobenius_norm",
    "extract_nonzero_fibers",
]

DENSE_CAP = 10_000_000  # tensor.py:42
_LIMIT = 1 << 63


class FormatError(ValueError):
    """Bad input data (coordinates out of range, duplicates, ragged arrays)."""


class ContractViolationError(RuntimeError):
    """Called outside the documented precondition (e.g. a train that is not
    orthonormal around the requested pivot)."""


def check_shape(shape) -> tuple[int, ...]:
    """Positive integer extents whose product stays below 2**63
    (tensor.py:47-67)."""
    items = tuple(shape)
    try:
        dims = tuple(operator.index(n) for n in items)
    except TypeError:
        raise TypeError(f"shape extents must be integers, got {items}") from None
    if not dims:
        raise ValueError("shape needs at least one mode")
    if min(dims) < 1:
        raise ValueError(f"shape extents must be positive, got {dims}")
    total = 1
    for n in dims:
        total *= n
        if total >= _LIMIT:
            raise ValueError(f"shape {dims} overflows 64-bit indexing")
    return dims


def size_of(shape) -> int:
    return math.prod(check_shape(shape))


def _c_strides(dims) -> np.ndarray:
    out = np.ones(len(dims), dtype=np.int64)
    acc = 1
    for k in range(len(dims) - 1, -1, -1):
        out[k] = acc
        acc *= dims[k]
    return out


def linearize(shape, coords) -> np.ndarray:
    """Row-major (last index fastest) linear index of each coordinate row."""
    dims = check_shape(shape)
    return np.asarray(coords, dtype=np.int64) @ _c_strides(dims)


def delinearize(shape, lin) -> np.ndarray:
    """Inverse of :func:`linearize`: ``(n,)`` linear indices -> ``(n, d)``."""
    dims = check_shape(shape)
    rem = np.asarray(lin, dtype=np.int64).copy()
    out = np.empty((rem.shape[0], len(dims)), dtype=np.int64)
    for k in range(len(dims) - 1, -1, -1):
        out[:, k] = rem % dims[k]
        rem //= dims[k]
    return out


class SparseTensor:
    """Immutable canonical COO tensor (reference tensor.py:103-197).

    Zeros are dropped, entries are stably sorted by C-order linear index and
    duplicate coordinates raise :class:`FormatError` (they are never summed).
    """

    __slots__ = ("shape", "coords", "values", "_lin", "_dev", "_pin", "_linq")

    def __init__(self, shape, coords, values):
        dims = check_shape(shape)
        d = len(dims)
        c = np.ascontiguousarray(coords, dtype=np.int64)
        v = np.ascontiguousarray(values, dtype=np.float64)
        if c.size == 0:
            c = c.reshape(0, d)
        if c.ndim != 2 or c.shape[1] != d:
            raise FormatError(f"coords must be (nnz, {d}), got {c.shape}")
        if v.shape != (c.shape[0],):
            raise FormatError(f"values must be ({c.shape[0]},), got {v.shape}")
        if c.shape[0]:
            lim = np.asarray(dims, dtype=np.int64)
            bad_rows = (c < 0).any(axis=1) | (c >= lim).any(axis=1)
            if bad_rows.any():
                first = int(np.argmax(bad_rows))
                raise FormatError(
                    f"coordinate {tuple(c[first])} out of range for shape {dims}")
        if not np.isfinite(v).all():
            raise FormatError("tensor values must be finite")
        nz = v != 0.0
        c, v = c[nz], v[nz]
        lin = c @ _c_strides(dims)
        order = np.argsort(lin, kind="stable")
        slin = lin[order]
        same = np.flatnonzero(slin[1:] == slin[:-1])
        if same.size:
            raise FormatError(f"duplicate coordinate {tuple(c[order[same[0] + 1]])}")
        c = np.ascontiguousarray(c[order])
        v = np.ascontiguousarray(v[order])
        c.setflags(write=False)
        v.setflags(write=False)
        slin = np.ascontiguousarray(slin)
        slin.setflags(write=False)
        object.__setattr__(self, "shape", dims)
        object.__setattr__(self, "coords", c)
        object.__setattr__(self, "values", v)
        # the canonical C-order linear index (the sort key above): the compact
        # form the COO travels to the device in (8 B per nonzero instead of 8d)
        object.__setattr__(self, "_lin", slin)
        object.__setattr__(self, "_dev", None)
        object.__setattr__(self, "_linq", None)
        object.__setattr__(self, "_pin", None)

    def __setattr__(self, name, value):
        raise AttributeError("SparseTensor is immutable")

    @classmethod
    def _from_canonical_device(cls, shape, coords_d, values_d) -> "SparseTensor":
        """A tensor whose canonical form (nonzero, C-order sorted, unique) was
        produced on the device (ftt_tensorize_matrix): the host arrays are a
        D2H copy and the device arrays stay cached -- no re-upload."""
        dims = check_shape(shape)
        c = np.ascontiguousarray(coords_d.cpu().numpy(), dtype=np.int64).reshape(-1, len(dims))
        v = np.ascontiguousarray(values_d.cpu().numpy(), dtype=np.float64)
        c.setflags(write=False)
        v.setflags(write=False)
        t = cls.__new__(cls)
        object.__setattr__(t, "shape", dims)
        object.__setattr__(t, "coords", c)
        object.__setattr__(t, "values", v)
        object.__setattr__(t, "_lin", None)
        object.__setattr__(t, "_dev", (coords_d, values_d, None, None))
        object.__setattr__(t, "_linq", None)
        object.__setattr__(t, "_pin", None)
        return t

    @property
    def ndim(self) -> int:
        return len(self.shape)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    @property
    def size(self) -> int:
        return math.prod(self.shape)

    def __repr__(self) -> str:
        return f"SparseTensor(shape={self.shape}, nnz={self.nnz})"

    @classmethod
    def from_dense(cls, a) -> "SparseTensor":
        a = np.ascontiguousarray(a, dtype=np.float64)
        where = np.argwhere(a != 0.0)
        return cls(a.shape, where, a[tuple(where.T)])

    def to_dense(self, cap: int | None = DENSE_CAP) -> np.ndarray:
        if cap is not None and self.size > cap:
            raise ValueError(f"dense size {self.size} exceeds cap {cap}; raise cap explicitly")
        out = np.zeros(self.size)
        out[linearize(self.shape, self.coords)] = self.values
        return out.reshape(self.shape)

    # -- device copy (host -> HBM once; reused by every GPU call on this tensor)
    # _dev = (coords or None, values, lin or None, values_ready event or None)
    def _pinned(self):
        pin = self._pin
        if pin is None:
            torch = nat.torch_mod()
            compact = self._lin is not None and self.nnz > 0
            src = self._lin if compact else self.coords
            pc = torch.empty(src.shape, dtype=torch.int64, pin_memory=True)
            pv = torch.empty(self.values.shape, dtype=torch.float64, pin_memory=True)
            pc.numpy()[...] = src
            pv.numpy()[...] = self.values
            pin = (pc, pv)
            object.__setattr__(self, "_pin", pin)
        return pin

    def _upload(self):
        """H2D of the canonical form: `lin` on the current stream (the index
        kernels start on it), the values on a side stream whose completion
        event the consumers wait for -- select_p's counts (which read only
        `lin`) overlap the values' transfer."""
        torch = nat.torch_mod()
        pin = self._pinned()
        compact = self._lin is not None and self.nnz > 0
        main = torch.cuda.current_stream()
        side = _side_stream()
        n = int(pin[0].shape[0])
        linq = None
        if compact and n >= _LIN_CHUNK_MIN:
            # large inputs: lin goes up in chunks on the side stream, each with
            # its event -- the first reader (select_p's forward counts,
            # ftt_set_lin_chunks) starts on the chunks present instead of
            # after the whole 8 B x nnz transfer
            lin = torch.empty(n, dtype=torch.int64, device="cuda")
            side.wait_stream(main)
            ends, evs = [], []
            with torch.cuda.stream(side):
                for j in range(_LIN_CHUNKS):
                    lo, hi = n * j // _LIN_CHUNKS, n * (j + 1) // _LIN_CHUNKS
                    lin[lo:hi].copy_(pin[0][lo:hi], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(side)
                    ends.append(hi)
                    evs.append(e)
            lin.record_stream(side)
            linq = (ends, evs)
        else:
            lin = pin[0].to("cuda", non_blocking=True)
            side.wait_stream(main)
        with torch.cuda.stream(side):
            v = pin[1].to("cuda", non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        v.record_stream(main)
        object.__setattr__(self, "_linq", linq)
        if compact:
            object.__setattr__(self, "_dev", (None, v, lin, ev))
        else:  # no canonical linear index on the host: these are the coordinates
            object.__setattr__(self, "_dev", (lin, v, None, ev))

    def _lin_arrived(self):
        """Make the current stream wait for a chunked `lin` upload (readers
        other than the fused fasttt call, which takes the chunk events)."""
        q = self._linq
        if q is not None:
            nat.torch_mod().cuda.current_stream().wait_event(q[1][-1])
            object.__setattr__(self, "_linq", None)

    def take_lin_chunks(self):
        """``(ends, events)`` of a chunked `lin` upload still in flight, or
        None; the caller takes over the waiting (ftt_set_lin_chunks)."""
        q = self._linq
        object.__setattr__(self, "_linq", None)
        return q

    def device_arrays(self):
        """``(coords, values)`` as CUDA tensors (cached).  The host side is
        staged once in pinned memory; what crosses PCIe is the canonical
        linear index (8 B per nonzero) and the values, and the coordinate
        rows are rebuilt on the device (``ftt_delinearize``) only when a
        caller needs them."""
        if self._dev is None:
            self._upload()
        self._lin_arrived()
        c, v, lin, ev = self._dev
        if ev is not None:
            nat.torch_mod().cuda.current_stream().wait_event(ev)
        if c is None:
            torch = nat.torch_mod()
            c = torch.empty(self.coords.shape, dtype=torch.int64, device="cuda")
            nat.check(nat.lib().ftt_delinearize(nat.context(), nat.ptr(lin), self.nnz, self.ndim,
                                                nat.i64_array(self.shape), nat.ptr(c)),
                      "ftt_delinearize")
        object.__setattr__(self, "_dev", (c, v, lin, None))
        return c, v

    def device_lin_values(self, keep_chunks=False):
        """``(lin, values, values_ready)``: the canonical linear index and the
        values on the device without the coordinate rows; `values_ready` is
        an event the consumer of `values` must wait for (or None).  With
        `keep_chunks` a chunked `lin` upload is left in flight for
        `take_lin_chunks`."""
        if self._dev is None:
            self._upload()
        if not keep_chunks:
            self._lin_arrived()
        c, v, lin, ev = self._dev
        if lin is None:
            lin = self.device_lin()
            c, v, lin, ev = self._dev
        return lin, v, ev

    def device_lin(self):
        """The canonical C-order linear index on the device (cached): the
        compact form the index kernels read (8 B per nonzero)."""
        if self._dev is None:
            self._upload()
        self._lin_arrived()
        lin = self._dev[2]
        if lin is None:
            c, v = self.device_arrays()
            torch = nat.torch_mod()
            lin = torch.empty(max(self.nnz, 1), dtype=torch.int64, device="cuda")
            nat.check(nat.lib().ftt_linearize(nat.context(), nat.ptr(c), self.nnz, self.ndim,
                                              nat.i64_array(self.shape), nat.ptr(lin)),
                      "ftt_linearize")
            object.__setattr__(self, "_dev", (c, v, lin, None))
        return lin

    @property
    def h2d_bytes(self) -> int:
        """Bytes device_arrays() moves host -> device."""
        lin = self._lin is not None and self.nnz > 0
        return int((self._lin.nbytes if lin else self.coords.nbytes) + self.values.nbytes)

    def drop_device_copy(self) -> None:
        """Forget the cached device arrays (the next GPU call re-uploads)."""
        object.__setattr__(self, "_dev", None)
        object.__setattr__(self, "_linq", None)


class FiberSet:
    """Nonzero fibers along one pivot mode, CSR-like (tensor.py:305-371)."""

    __slots__ = ("shape", "pivot", "fixed_coords", "indptr", "pivot_index", "values", "_dev")

    def __init__(self, shape, pivot, fixed_coords, indptr, pivot_index, values, _dev=None):
        dims = check_shape(shape)
        d = len(dims)
        if not 0 <= pivot < d:
            raise ValueError(f"pivot {pivot} out of range for {d} modes")
        fixed_coords = np.ascontiguousarray(fixed_coords, dtype=np.int64)
        indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        pivot_index = np.ascontiguousarray(pivot_index, dtype=np.int64)
        values = np.ascontiguousarray(values, dtype=np.float64)
        # the reference counts fibers as 0 when the fixed tuple is empty
        # (d = 1), so its single-fiber output fails the indptr check below
        r = fixed_coords.shape[0] if fixed_coords.size else 0
        fixed_coords = fixed_coords.reshape(r, d - 1)
        if indptr.shape != (r + 1,) or indptr[0] != 0 or indptr[-1] != values.shape[0]:
            raise ValueError("inconsistent fiber index pointers")
        if r and np.any(np.diff(indptr) < 1):
            raise ValueError("every stored fiber must hold at least one nonzero")
        if r > 1:
            rest = dims[:pivot] + dims[pivot + 1:]
            keys = linearize(rest, fixed_coords)
            if np.any(np.diff(keys) <= 0):
                raise ValueError("fixed tuples must be strictly increasing")
        for arr in (fixed_coords, indptr, pivot_index, values):
            arr.setflags(write=False)
        object.__setattr__(self, "shape", dims)
        object.__setattr__(self, "pivot", int(pivot))
        object.__setattr__(self, "fixed_coords", fixed_coords)
        object.__setattr__(self, "indptr", indptr)
        object.__setattr__(self, "pivot_index", pivot_index)
        object.__setattr__(self, "values", values)
        object.__setattr__(self, "_dev", _dev)

    def __setattr__(self, name, value):
        raise AttributeError("FiberSet is immutable")

    @property
    def num_fibers(self) -> int:
        return int(self.fixed_coords.shape[0])

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def __iter__(self):
        for i in range(self.num_fibers):
            lo, hi = self.indptr[i], self.indptr[i + 1]
            yield tuple(self.fixed_coords[i]), (self.pivot_index[lo:hi], self.values[lo:hi])

    def to_tensor(self) -> SparseTensor:
        d = len(self.shape)
        rest = [k for k in range(d) if k != self.pivot]
        owner = np.repeat(np.arange(self.num_fibers), np.diff(self.indptr))
        coords = np.empty((self.nnz, d), dtype=np.int64)
        coords[:, rest] = self.fixed_coords[owner]
        coords[:, self.pivot] = self.pivot_index
        return SparseTensor(self.shape, coords, self.values)


_SIDE = {}


_LIN_CHUNK_MIN = 1 << 21  # nonzeros from which `lin` is uploaded in chunks
_LIN_CHUNKS = 4


def _side_stream():
    """One side stream per device for the values' H2D copy."""
    torch = nat.torch_mod()
    dev = torch.cuda.current_device()
    st = _SIDE.get(dev)
    if st is None:
        st = _SIDE[dev] = torch.cuda.Stream(dev)
    return st


def frobenius_norm(t) -> float:
    """Frobenius norm (tensor.py:298-302), reduced on the GPU."""
    torch = nat.torch_mod()
    if isinstance(t, SparseTensor):
        if t.nnz == 0:
            return 0.0
        _, v = t.device_arrays()
    else:
        v = torch.from_numpy(np.ascontiguousarray(t, dtype=np.float64).ravel()).to("cuda")
    return float(np.sqrt(device_dot(v, None)))


def device_dot(x, y) -> float:
    out = nat.ctypes.c_double(0.0)
    nat.check(nat.lib().ftt_dot(nat.context(), int(x.numel()), nat.ptr(x), nat.ptr(y),
                                nat.ctypes.byref(out)), "ftt_dot")
    return float(out.value)


class DeviceFibers:
    """Device-resident result of the fiber extraction (all int64/float64)."""

    __slots__ = ("dims", "pivot", "R", "nnz", "fixed_lin", "indptr", "fiber_of",
                 "pivot_index", "values")

    def __init__(self, dims, pivot, R, nnz, fixed_lin, indptr, fiber_of, pivot_index, values):
        self.dims = dims
        self.pivot = pivot
        self.R = R
        self.nnz = nnz
        self.fixed_lin = fixed_lin
        self.indptr = indptr
        self.fiber_of = fiber_of
        self.pivot_index = pivot_index
        self.values = values

    def rest_stride(self, k: int) -> int:
        """Stride of mode k inside the fixed-tuple linear index."""
        rest = [self.dims[j] for j in range(len(self.dims)) if j != self.pivot]
        col = k if k < self.pivot else k - 1
        return math.prod(rest[col + 1:])

    def fixed_coords_host(self) -> np.ndarray:
        torch = nat.torch_mod()
        d = len(self.dims)
        out = torch.empty((max(d - 1, 0), max(self.R, 0)), dtype=torch.int64, device="cuda")
        ctx = nat.context()
        for k in range(d):
            if k == self.pivot:
                continue
            col = k if k < self.pivot else k - 1
            if self.R:
                nat.check(nat.lib().ftt_mode_index(ctx, nat.ptr(self.fixed_lin), self.R,
                                                   self.rest_stride(k), self.dims[k],
                                                   nat.ptr(out[col])), "ftt_mode_index")
        return np.ascontiguousarray(out.cpu().numpy().T)


def fibers_device(dims, pivot, coords_d, values_d, nnz, lin_d=None) -> DeviceFibers:
    """ftt_extract_fibers on device arrays (ftt_extract_fibers_lin when the
    canonical linear index is given)."""
    torch = nat.torch_mod()
    d = len(dims)
    cap = max(nnz, 1)
    fixed_lin = torch.empty(cap, dtype=torch.int64, device="cuda")
    indptr = torch.empty(cap + 1, dtype=torch.int64, device="cuda")
    fiber_of = torch.empty(cap, dtype=torch.int64, device="cuda")
    pidx = torch.empty(cap, dtype=torch.int64, device="cuda")
    vals = torch.empty(cap, dtype=torch.float64, device="cuda")
    R = nat.ctypes.c_int64(0)
    if lin_d is not None:
        nat.check(nat.lib().ftt_extract_fibers_lin(
            nat.context(), nat.ptr(lin_d), nat.ptr(values_d), int(nnz), d, nat.i64_array(dims),
            int(pivot), nat.ptr(fixed_lin), nat.ptr(indptr), nat.ptr(fiber_of), nat.ptr(pidx),
            nat.ptr(vals), nat.ctypes.byref(R)), "ftt_extract_fibers_lin")
    else:
        nat.check(nat.lib().ftt_extract_fibers(
            nat.context(), nat.ptr(coords_d), nat.ptr(values_d), int(nnz), d, nat.i64_array(dims),
            int(pivot), nat.ptr(fixed_lin), nat.ptr(indptr), nat.ptr(fiber_of), nat.ptr(pidx),
            nat.ptr(vals), nat.ctypes.byref(R)), "ftt_extract_fibers")
    R = int(R.value)
    return DeviceFibers(tuple(dims), int(pivot), R, int(nnz), fixed_lin[:R], indptr[:R + 1],
                        fiber_of[:nnz], pidx[:nnz], vals[:nnz])


def extract_nonzero_fibers(t: SparseTensor, pivot: int) -> FiberSet:
    """Group nonzeros into mode-``pivot`` fibers (tensor.py:374-403) on the
    GPU: one radix sort of ``lin(fixed) * n_p + i_p`` plus a segmented scan."""
    d = t.ndim
    if not 0 <= pivot < d:
        raise ValueError(f"pivot {pivot} out of range for {d} modes")
    if t.nnz == 0:
        return FiberSet(t.shape, pivot, np.zeros((0, max(d - 1, 0)), np.int64),
                        np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    lin, v, ev = t.device_lin_values()
    if ev is not None:
        nat.torch_mod().cuda.current_stream().wait_event(ev)
    df = fibers_device(t.shape, pivot, None, v, t.nnz, lin_d=lin)
    fixed = df.fixed_coords_host() if d > 1 else np.zeros((df.R, 0), np.int64)
    return FiberSet(t.shape, pivot, fixed, df.indptr.cpu().numpy(), df.pivot_index.cpu().numpy(),
                    df.values.cpu().numpy(), _dev=df)
