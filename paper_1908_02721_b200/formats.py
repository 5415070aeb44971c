"""Input side of the decomposition path: COO text tensors and MatrixMarket
matrices (reference formats.py:38-127).

Text formats are 1-based on disk and 0-based in memory.  ``ingest_coo``
parses well-formed files in native code (``ftt_parse_coo_text``, one pass,
strtoll/strtod) -- the reference reads them with a per-line Python loop; on
the first line the fast path rejects, the file is re-read with the
reference's own loop so every error carries the reference's exact
``FormatError`` text.  ``write_coo`` prints 17 significant digits so a
write/read round trip is bit-exact.
"""

from __future__ import annotations

import ctypes
import warnings

import numpy as np

from . import _native as nat
from .coo import FormatError, SparseTensor, check_shape

__all__ = ["write_coo", "ingest_coo", "ingest_matrix_market"]


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


def _native_parse(path):
    """(dims, coords, values) from the native reader, or None when it
    rejects the file (the reference loop then reports the error)."""
    lib = nat.lib()
    d = ctypes.c_int32(0)
    dims = (ctypes.c_int64 * 32)()
    nnz = ctypes.c_int64(0)
    cptr = ctypes.POINTER(ctypes.c_int64)()
    vptr = ctypes.POINTER(ctypes.c_double)()
    bad = ctypes.c_int64(0)
    st = lib.ftt_parse_coo_text(str(path).encode(), ctypes.byref(d), dims, ctypes.byref(nnz),
                                ctypes.byref(cptr), ctypes.byref(vptr), ctypes.byref(bad))
    if st != nat.FTT_OK:
        return None
    try:
        n, dd = int(nnz.value), int(d.value)
        coords = np.ctypeslib.as_array(cptr, shape=(max(n * dd, 1),))[: n * dd].copy()
        values = np.ctypeslib.as_array(vptr, shape=(max(n, 1),))[:n].copy()
    finally:
        lib.ftt_free_host(cptr)
        lib.ftt_free_host(vptr)
    return tuple(int(x) for x in dims[:dd]), coords.reshape(n, dd), values


def _ingest_coo_reference(path) -> SparseTensor:
    """The reference's line loop (formats.py:47-100), for its error texts."""
    with open(path, "r", encoding="ascii") as fh:
        lines = fh.readlines()
    if not lines:
        raise FormatError(f"{path}: empty file, missing shape header")
    head = lines[0].split()
    if len(head) < 3 or head[0] != "#" or head[1] != "shape":
        raise FormatError(f"{path}:1: expected header '# shape n1 ... nd'")
    try:
        dims = check_shape(int(tok) for tok in head[2:])
    except ValueError as exc:
        raise FormatError(f"{path}:1: bad shape header: {exc}") from None
    d = len(dims)
    coords, values = [], []
    for lineno, line in enumerate(lines[1:], start=2):
        tok = line.split()
        if not tok:
            continue
        if len(tok) != d + 1:
            raise FormatError(f"{path}:{lineno}: expected {d} indices and a value, "
                              f"got {len(tok)} fields")
        try:
            idx = [int(s) for s in tok[:d]]
            val = float(tok[d])
        except ValueError:
            raise FormatError(f"{path}:{lineno}: unparsable entry {line.strip()!r}") from None
        for k, i in enumerate(idx):
            if not 1 <= i <= dims[k]:
                raise FormatError(f"{path}:{lineno}: index {i} out of range 1..{dims[k]} "
                                  f"in mode {k + 1}")
        if not np.isfinite(val):
            raise FormatError(f"{path}:{lineno}: non-finite value {tok[d]}")
        coords.append([i - 1 for i in idx])
        values.append(val)
    return _finish(path, dims, np.asarray(coords, np.int64).reshape(len(values), d), values)


def _finish(path, dims, coords, values) -> SparseTensor:
    if len(values) == 0:
        warnings.warn(f"{path}: no entries, reading the zero tensor", stacklevel=3)
    try:
        return SparseTensor(dims, coords, values)
    except FormatError as exc:
        raise FormatError(f"{path}: {exc}") from None


def ingest_coo(path) -> SparseTensor:
    """Read the COO text format written by :func:`write_coo`
    (formats.py:47-100): ``# shape n1 ... nd`` header, then ``d`` 1-based
    indices and a value per nonempty line; duplicates are an error; an
    empty entry list yields the zero tensor with a warning."""
    fast = _native_parse(path)
    if fast is None:
        return _ingest_coo_reference(path)
    dims, coords, values = fast
    try:
        dims = check_shape(dims)
    except ValueError:
        return _ingest_coo_reference(path)
    return _finish(path, dims, coords, values)


def ingest_matrix_market(path):
    """Coordinate-format real MatrixMarket, ``general`` or ``symmetric``
    (formats.py:103-127); returns a ``scipy.sparse.coo_matrix``."""
    import scipy.io
    import scipy.sparse

    with open(path, "r", encoding="ascii") as fh:
        banner = fh.readline().split()
    if len(banner) != 5 or banner[0] != "%%MatrixMarket":
        raise FormatError(f"{path}:1: not a MatrixMarket file")
    obj, fmt, field, symmetry = (s.lower() for s in banner[1:])
    if obj != "matrix":
        raise FormatError(f"{path}: unsupported MatrixMarket object {obj!r}")
    if fmt != "coordinate":
        raise FormatError(f"{path}: unsupported MatrixMarket format {fmt!r} (need coordinate)")
    if field != "real":
        raise FormatError(f"{path}: unsupported MatrixMarket field {field!r} (need real)")
    if symmetry not in ("general", "symmetric"):
        raise FormatError(f"{path}: unsupported MatrixMarket symmetry {symmetry!r} "
                          "(need general or symmetric)")
    try:
        m = scipy.io.mmread(path)
    except Exception as exc:  # noqa: BLE001
        raise FormatError(f"{path}: {exc}") from None
    return scipy.sparse.coo_matrix(m, dtype=np.float64)
