"""Truncated SVD and economic QR on the GPU (drop-in for linalg.py).

The factorizations are libfasttt_b200 kernels (blocked Householder QR and
one-sided block Jacobi, ftt_qr_f64 / ftt_svd_f64); only the scalar tail rule
that turns singular values into a rank -- a scan over ``min(m, n)`` numbers
the reference also runs on the host (linalg.py:89-100) -- is Python.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat

__all__ = ["SVDResult", "QRResult", "svd_truncate_delta", "svd_truncate_rank", "qr_economic",
           "tail_rank", "tail_error"]

_EPS = float(np.finfo(np.float64).eps)


@dataclass(frozen=True, eq=False)
class SVDResult:
    """``m ~= u @ diag(s) @ vt``; ``trunc_error`` = norm of the discarded part."""

    u: np.ndarray
    s: np.ndarray
    vt: np.ndarray
    rank: int
    trunc_error: float


@dataclass(frozen=True, eq=False)
class QRResult:
    """``m = q @ r`` with ``diag(r) >= 0``."""

    q: np.ndarray
    r: np.ndarray


def tail_rank(s: np.ndarray, delta: float, shape, rest2: float = 0.0) -> int:
    """Smallest kept rank whose discarded tail has ``sum(s[r:]**2) <= delta**2``;
    ``delta == 0`` keeps ``s >= max(shape) * eps * s[0]`` (linalg.py:89-99).
    ``rest2`` is the certified energy beyond the returned values (low-rank
    path; 0 for a full SVD, which makes this the reference rule verbatim)."""
    if delta == 0.0:
        if s.size == 0 or s[0] == 0.0:
            return 0
        return int(np.count_nonzero(s >= max(shape) * _EPS * s[0]))
    sq = s * s
    tails = np.concatenate([np.cumsum(sq[::-1])[::-1], [0.0]])
    if rest2:
        tails = tails + rest2
    return int(np.argmax(tails <= delta * delta))


def tail_error(s: np.ndarray, rank: int, rest2: float = 0.0) -> float:
    sq = s * s
    return float(np.sqrt(max(float(np.sum(sq[rank:])) + rest2, 0.0)))


LOWRANK_MIN = 16        # smaller operands: the full SVD is already cheap


def lowrank_k(min_dim: int, hint) -> int:
    """Sketch width for the certified low-rank path (0 = do not try)."""
    if min_dim < LOWRANK_MIN:
        return 0
    k = 32 if hint is None else max(16, 2 * int(hint) + 8)
    k = (k + 7) // 8 * 8
    # narrow operands (<= 64 columns) also take the sketch when it is narrower:
    # the full path's column-sequential TSQR + Jacobi cost grows with the
    # width, the sketch path's with the (certified) rank
    # sketches wider than 64 columns (bonds of rank > 28) belong to operands
    # with genuine tails (configs 3 and 4): measured always rejected there, so
    # the attempt is skipped
    if k > 64:
        return 0
    if k < min_dim and (2 * k <= min_dim or min_dim <= 64):
        return k
    return 0


def dev_svd_values_lowrank(buf, m: int, n: int, ld: int, row_major: bool, k: int,
                           delta2: float):
    """Phase 1 of the certified low-rank path: (s[k], rest2, accepted) with
    accepted 2 = residual below full-SVD noise, 1 = rest2 <= 1e-6 delta^2
    (interval-certified use only), 0 = rejected."""
    s = np.zeros(k)
    rest2 = nat.ctypes.c_double(0.0)
    acc = nat.ctypes.c_int32(0)
    nat.check(nat.lib().ftt_svd_lowrank_f64(
        nat.context(), int(m), int(n), nat.ptr(buf), int(ld), int(bool(row_major)), int(k),
        float(delta2), s.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_double)),
        nat.ctypes.byref(rest2), nat.ctypes.byref(acc)), "ftt_svd_lowrank_f64")
    return s, float(rest2.value), int(acc.value)


def dev_svd_truncate(buf, m: int, n: int, ld: int, row_major: bool, delta, hint=None,
                     interval_ok: bool = False):
    """Phase 1 for a truncation step: (s, rest2). Tries the certified
    low-rank path when delta > 0, else (or on rejection) the full SVD.

    The low-rank values bound every true tail sum of the operand inside
    [tail_B(r), tail_B(r) + rest2] (Ky Fan: A^T A = B^T B + E^T E with
    ||E||_F^2 = rest2).  A residual above the full-SVD noise level is still
    used (``interval_ok``, static budgets) when the rank rule gives the same
    answer at both ends of that interval -- then the decision is the exact
    arithmetic one, like the reference's."""
    if delta is not None and delta > 0.0:
        k = lowrank_k(min(m, n), hint)
        if k:
            s, rest2, acc = dev_svd_values_lowrank(buf, m, n, ld, row_major, k, delta * delta)
            if acc == 2:
                return s, rest2
            if acc == 1 and interval_ok:
                shape = (m, n)
                if tail_rank(s, delta, shape, 0.0) == tail_rank(s, delta, shape, rest2):
                    return s, rest2
    return dev_svd_values(buf, m, n, ld, row_major), 0.0


def _check_matrix(m) -> np.ndarray:
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2:
        raise ValueError(f"expected a matrix, got ndim={m.ndim}")
    if not np.isfinite(m).all():
        raise ValueError("matrix entries must be finite")
    return m


def dev_svd_values(buf, m: int, n: int, ld: int, row_major: bool) -> np.ndarray:
    """Phase 1 of the device SVD: singular values (descending, host array)."""
    k = min(m, n)
    s = np.zeros(max(k, 1))
    nat.check(nat.lib().ftt_svd_f64(nat.context(), int(m), int(n), nat.ptr(buf), int(ld),
                                    int(bool(row_major)),
                                    s.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_double))),
              "ftt_svd_f64")
    return s[:k]


def dev_svd_vectors(m: int, n: int, rank: int, u_row_major: bool, v_row_major: bool,
                    scale_v: bool):
    """Phase 2: U (m x rank) and V = vt.T (n x rank) of the last phase 1 as
    torch tensors whose buffers are row- or column-major per flag."""
    torch = nat.torch_mod()
    if u_row_major:
        U = torch.empty((m, rank), dtype=torch.float64, device="cuda")
        ldu = rank
    else:
        U = torch.empty((rank, m), dtype=torch.float64, device="cuda")
        ldu = m
    if v_row_major:
        V = torch.empty((n, rank), dtype=torch.float64, device="cuda")
        ldv = rank
    else:
        V = torch.empty((rank, n), dtype=torch.float64, device="cuda")
        ldv = n
    if rank:
        nat.check(nat.lib().ftt_svd_vectors(nat.context(), int(rank), nat.ptr(U), max(ldu, 1),
                                            int(u_row_major), nat.ptr(V), max(ldv, 1),
                                            int(v_row_major), int(bool(scale_v))),
                  "ftt_svd_vectors")
    return U, V


def _svd_host_api(m, rank_of):
    m = _check_matrix(m)
    rows, cols = m.shape
    torch = nat.torch_mod()
    dm = torch.from_numpy(np.ascontiguousarray(m)).to("cuda")
    s = dev_svd_values(dm, rows, cols, max(cols, 1), True)
    rank = rank_of(s, m.shape)
    err = tail_error(s, rank)
    if rank == 0:
        return SVDResult(u=np.zeros((rows, 0)), s=np.zeros(0), vt=np.zeros((0, cols)), rank=0,
                         trunc_error=err)
    U, V = dev_svd_vectors(rows, cols, rank, True, False, False)
    return SVDResult(u=U.cpu().numpy(), s=s[:rank].copy(), vt=V.cpu().numpy(), rank=rank,
                     trunc_error=err)


def svd_truncate_delta(m, delta: float) -> SVDResult:
    """Truncated SVD keeping the smallest rank whose tail is within ``delta``
    (linalg.py:75-105)."""
    if delta < 0:
        _check_matrix(m)
        raise ValueError(f"delta must be nonnegative, got {delta}")
    return _svd_host_api(m, lambda s, shape: tail_rank(s, delta, shape))


def svd_truncate_rank(m, r: int) -> SVDResult:
    """Best approximation of rank ``min(r, min(m.shape))`` (linalg.py:108-125)."""
    if r < 0:
        _check_matrix(m)
        raise ValueError(f"target rank must be nonnegative, got {r}")
    return _svd_host_api(m, lambda s, shape: int(min(r, min(shape))))


def qr_economic(m) -> QRResult:
    """Reduced Householder QR with ``diag(r) >= 0`` (linalg.py:128-140)."""
    m = _check_matrix(m)
    rows, cols = m.shape
    from .trains import dev_qr

    torch = nat.torch_mod()
    k = min(rows, cols)
    if k == 0:
        return QRResult(q=np.zeros((rows, 0)), r=np.zeros((0, cols)))
    # column-major m == row-major m.T
    dmT = torch.from_numpy(np.ascontiguousarray(m.T)).to("cuda")
    Q, R = dev_qr(dmT, rows, cols, rows)
    return QRResult(q=np.ascontiguousarray(Q.cpu().numpy().T), r=np.ascontiguousarray(R.cpu().numpy().T))
