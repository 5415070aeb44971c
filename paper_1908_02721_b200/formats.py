"""Input side of the decomposition path: COO text tensors and MatrixMarket
matrices (reference formats.py:38-127).

Text formats are 1-based on disk and 0-based in memory.  Both readers are
native (csrc/ftt_io.cu): ``ftt_parse_coo_text`` decides everything the
reference's ``ingest_coo`` decides -- line and token splitting, Python's
int()/float() literal grammar, the order of its checks -- and reports a
rejected file as an error record that this module only words into the
reference's ``FormatError`` text.  ``ftt_parse_mm_text`` classifies the
MatrixMarket banner and reads strict ``real general|symmetric`` bodies; a
body it does not accept goes to ``scipy.io.mmread``, the library the
reference reads with, for its result or exception text.  ``write_coo``
prints 17 significant digits so a write/read round trip is bit-exact.
"""

from __future__ import annotations

import ctypes
import warnings

import numpy as np

from . import _native as nat
from .coo import FormatError, SparseTensor, check_shape

__all__ = ["write_coo", "ingest_coo", "ingest_matrix_market"]

_MAX_MODES = 4096

# error kinds of ftt_parse_coo_text (include/fasttt_b200.h)
(_IO, _EMPTY, _HEADER, _SHAPE, _FIELDS, _UNPARSABLE, _RANGE, _NONFINITE,
 _NONASCII) = range(1, 10)
# banner classes of ftt_parse_mm_text
_MM_NOT_MM, _MM_OBJECT, _MM_FORMAT, _MM_FIELD, _MM_SYMMETRY, _MM_GENERAL, _MM_SYMMETRIC = \
    range(1, 8)


class _CooError(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("mode", ctypes.c_int32), ("line", ctypes.c_int64),
                ("count", ctypes.c_int64), ("text", ctypes.POINTER(ctypes.c_char)),
                ("text_len", ctypes.c_int64)]


def write_coo(t: SparseTensor, path) -> None:
    """Shape header, then one line per nonzero with 1-based coordinates."""
    d = t.ndim
    with open(path, "w", encoding="ascii") as fh:
        fh.write("# shape " + " ".join(str(n) for n in t.shape) + "\n")
        if t.nnz:
            cols = [np.char.mod("%d", t.coords[:, k] + 1) for k in range(d)]
            vals = [f"{v:.17g}" for v in t.values.tolist()]
            rows = [" ".join(parts) for parts in zip(*cols, vals)]
            fh.write("\n".join(rows) + "\n")


def _take_host(ptr, n, dtype):
    """Copy ``n`` items out of a malloc'd native buffer and free it."""
    try:
        if not ptr or n == 0:
            return np.zeros(0, dtype=dtype)
        return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)
    finally:
        if ptr:
            nat.lib().ftt_free_host(ptr)


def _shape_header_message(header: str) -> str:
    """The ValueError text int()/check_shape give for the header's extents
    (the native reader found that they fail)."""
    try:
        check_shape(int(tok) for tok in header.split()[2:])
    except ValueError as exc:
        return str(exc)
    return f"more than {_MAX_MODES} modes"


def _coo_error(path, err: _CooError, dims):
    kind = err.kind
    text = ctypes.string_at(err.text, err.text_len).decode("ascii") if err.text else ""
    if err.text:
        nat.lib().ftt_free_host(err.text)
    line = int(err.line)
    where = f"{path}:{line}"
    if kind == _IO:
        with open(path, "rb"):
            pass
        return OSError(f"{path}: unreadable")
    if kind == _NONASCII:
        return UnicodeDecodeError("ascii", bytes([err.mode]), 0, 1, "ordinal not in range(128)")
    if kind == _EMPTY:
        return FormatError(f"{path}: empty file, missing shape header")
    if kind == _HEADER:
        return FormatError(f"{path}:1: expected header '# shape n1 ... nd'")
    if kind == _SHAPE:
        return FormatError(f"{path}:1: bad shape header: {_shape_header_message(text)}")
    if kind == _FIELDS:
        return FormatError(f"{where}: expected {len(dims)} indices and a value, "
                           f"got {int(err.count)} fields")
    if kind == _UNPARSABLE:
        return FormatError(f"{where}: unparsable entry {text.strip()!r}")
    if kind == _RANGE:
        k = int(err.mode)
        return FormatError(f"{where}: index {int(text)} out of range 1..{dims[k]} in mode {k + 1}")
    if kind == _NONFINITE:
        return FormatError(f"{where}: non-finite value {text}")
    return FormatError(f"{path}: unreadable COO text ({nat.last_error()})")


def ingest_coo(path) -> SparseTensor:
    """Read the COO text format written by :func:`write_coo`
    (formats.py:47-100): ``# shape n1 ... nd`` header, then ``d`` 1-based
    indices and a value per nonempty line; duplicates are an error; an
    empty entry list yields the zero tensor with a warning."""
    lib = nat.lib()
    d = ctypes.c_int32(0)
    dims_buf = (ctypes.c_int64 * _MAX_MODES)()
    nnz = ctypes.c_int64(0)
    cptr = ctypes.POINTER(ctypes.c_int64)()
    vptr = ctypes.POINTER(ctypes.c_double)()
    err = _CooError()
    st = lib.ftt_parse_coo_text(str(path).encode(), _MAX_MODES, ctypes.byref(d), dims_buf,
                                ctypes.byref(nnz), ctypes.byref(cptr), ctypes.byref(vptr),
                                ctypes.byref(err))
    dims = tuple(int(x) for x in dims_buf[: d.value])
    if st == nat.FTT_ERR_OOM:
        raise MemoryError(nat.last_error())
    if st != nat.FTT_OK:
        raise _coo_error(path, err, dims)
    n = int(nnz.value)
    coords = _take_host(cptr, n * len(dims), np.int64).reshape(n, len(dims))
    values = _take_host(vptr, n, np.float64)
    if n == 0:
        warnings.warn(f"{path}: no entries, reading the zero tensor", stacklevel=2)
    try:
        return SparseTensor(dims, coords, values)
    except FormatError as exc:
        raise FormatError(f"{path}: {exc}") from None


def ingest_matrix_market(path):
    """Coordinate-format real MatrixMarket, ``general`` or ``symmetric``
    (formats.py:103-127); returns a ``scipy.sparse.coo_matrix``."""
    import scipy.io
    import scipy.sparse

    lib = nat.lib()
    banner = ctypes.c_int32(0)
    shape = (ctypes.c_int64 * 2)()
    nnz = ctypes.c_int64(0)
    rp = ctypes.POINTER(ctypes.c_int64)()
    cp = ctypes.POINTER(ctypes.c_int64)()
    vp = ctypes.POINTER(ctypes.c_double)()
    st = lib.ftt_parse_mm_text(str(path).encode(), ctypes.byref(banner), shape,
                               ctypes.byref(nnz), ctypes.byref(rp), ctypes.byref(cp),
                               ctypes.byref(vp))
    if st == nat.FTT_ERR_OOM:
        raise MemoryError(nat.last_error())
    b = banner.value
    if b not in (_MM_GENERAL, _MM_SYMMETRIC):
        with open(path, "r", encoding="ascii") as fh:  # decode errors as the reference's
            words = fh.readline().split()
        if b == _MM_NOT_MM or len(words) != 5:
            raise FormatError(f"{path}:1: not a MatrixMarket file")
        what = {_MM_OBJECT: ("object", 1, ""), _MM_FORMAT: ("format", 2, " (need coordinate)"),
                _MM_FIELD: ("field", 3, " (need real)"),
                _MM_SYMMETRY: ("symmetry", 4, " (need general or symmetric)")}[b]
        raise FormatError(f"{path}: unsupported MatrixMarket {what[0]} "
                          f"{words[what[1]].lower()!r}{what[2]}")
    if st == nat.FTT_OK:
        n = int(nnz.value)
        rows = _take_host(rp, n, np.int64)
        cols = _take_host(cp, n, np.int64)
        vals = _take_host(vp, n, np.float64)
        return scipy.sparse.coo_matrix((vals, (rows, cols)), shape=(int(shape[0]), int(shape[1])),
                                       dtype=np.float64)
    # a body outside the strict grammar: the library reader decides
    try:
        m = scipy.io.mmread(path)
    except Exception as exc:  # noqa: BLE001
        raise FormatError(f"{path}: {exc}") from None
    return scipy.sparse.coo_matrix(m, dtype=np.float64)
