"""Test-only helpers the reference's own unit tests import from ``sparsett``
but that are not on the decomposition path (so the product package does not
export them): dense TT contraction, the classical TT-SVD oracle, the
quasi-permutation recogniser and the dense materialisation of a structured
train.  Plain numpy, written for this test suite; each cites the reference
function whose contract it restates.  Nothing under paper_1908_02721_b200/
imports this module.
"""

from __future__ import annotations

import math

import numpy as np

import paper_1908_02721_b200 as ft


def rand_sparse(rng: np.random.Generator, shape, density: float) -> ft.SparseTensor:
    """Seeded distinct coordinates with nonzero U(-1, 1) values (the recipe of
    the reference's tests/conftest.py:10-17)."""
    size = math.prod(shape)
    nnz = int(density * size)
    lin = np.sort(rng.permutation(size)[:nnz].astype(np.int64))
    vals = rng.uniform(-1.0, 1.0, nnz)
    vals[vals == 0.0] = 0.5
    coords = np.stack(np.unravel_index(lin, shape), axis=1).astype(np.int64)
    return ft.SparseTensor(shape, coords.reshape(nnz, len(shape)), vals)


def tt_to_full(t: ft.TTTensor) -> np.ndarray:
    """Dense tensor of a train (ttformat.py tt_to_full): left-to-right
    contraction of the cores."""
    acc = np.ones((1, 1))
    dims = []
    for c in t.cores:
        c = np.asarray(c, dtype=np.float64)
        r0, n, r1 = c.shape
        acc = (acc @ c.reshape(r0, n * r1)).reshape(-1, r1)
        dims.append(n)
    return acc.reshape(dims)


def _tail_rank(s: np.ndarray, delta: float) -> int:
    # smallest r whose discarded tail sum_{i >= r} s_i^2 <= delta^2
    tail = np.concatenate([np.cumsum((s ** 2)[::-1])[::-1], [0.0]])
    return int(np.argmax(tail <= delta * delta))


def tt_svd(a: np.ndarray, eps: float) -> ft.TTTensor:
    """Classical TT-SVD with per-step budget eps / sqrt(d-1) * ||a||_F
    (ttsvd.py:23-48), LAPACK gesdd per unfolding."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    dims = a.shape
    d = a.ndim
    if d == 1:
        return ft.TTTensor([a.reshape(1, -1, 1)])
    delta = eps / math.sqrt(d - 1) * float(np.linalg.norm(a.ravel()))
    cores, c, r = [], a, 1
    for k in range(d - 1):
        m = c.reshape(r * dims[k], -1)
        if not np.any(m):
            return ft.tt_zero(dims)
        u, s, vt = np.linalg.svd(m, full_matrices=False)
        rank = _tail_rank(s, delta)
        if rank == 0:
            return ft.tt_zero(dims)
        cores.append(u[:, :rank].reshape(r, dims[k], rank))
        c = s[:rank, None] * vt[:rank]
        r = rank
    cores.append(c.reshape(r, dims[-1], 1))
    return ft.TTTensor(cores)


def as_quasi_perm(m):
    """QuasiPermMatrix if every column of ``m`` holds exactly one entry and
    it equals 1.0, else None (ttformat.py:266-278)."""
    if isinstance(m, ft.QuasiPermMatrix):
        return m
    m = np.asarray(m, dtype=np.float64)
    nz = m != 0.0
    if np.any(nz.sum(axis=0) != 1):
        return None
    rows = np.argmax(nz, axis=0)
    if m.shape[1] and not np.all(m[rows, np.arange(m.shape[1])] == 1.0):
        return None
    return ft.QuasiPermMatrix(m.shape[0], m.shape[1], rows.astype(np.int64))


def structured_to_tt(s: ft.StructuredTT) -> ft.TTTensor:
    """Explicit dense cores of the exact structured train
    (ttformat.py:368-402): interior bonds R, 0/1 side cores on the fiber
    diagonal, the pivot core holding each fiber's values."""
    d, r, dims = s.ndim, s.num_fibers, s.shape
    if r == 0:
        return ft.tt_zero(dims)
    ids = np.arange(r)
    f = s.fibers
    cores = []
    for k in range(d):
        r0 = r if k > 0 else 1
        r1 = r if k < d - 1 else 1
        core = np.zeros((r0, dims[k], r1))
        if k == s.pivot:
            owner = np.repeat(ids, np.diff(f.indptr))
            core[owner if k > 0 else 0, f.pivot_index, owner if k < d - 1 else 0] = f.values
        else:
            core[ids if k > 0 else 0, s.mode_index(k), ids if k < d - 1 else 0] = 1.0
        cores.append(core)
    return ft.TTTensor(cores)


def modeled_cost(shape, pivot, rt, r, c=1.0):
    """The pipeline cost model (fasttt.py:456-481) restated independently:
    pivot-core SVD, the outward SVDs right of the pivot, the left ones."""
    d = len(shape)
    frt = (1,) + tuple(rt) + (1,)
    fr = (1,) + tuple(r) + (1,)

    def f(m, n):
        return m * n * min(m, n)

    p = pivot + 1
    total = f(frt[p - 1] * shape[p - 1], frt[p])
    total += sum(f(fr[i - 1] * shape[i - 1], frt[i]) for i in range(p + 1, d))
    total += sum(f(frt[i - 1], shape[i - 1] * fr[i]) for i in range(2, p + 1))
    return c * total


def brute_select(a: ft.SparseTensor, target=None) -> int:
    """select_p by enumeration: distinct fixed tuples from a Python set per
    pivot, the upper bond bounds of fasttt.py:484-497, first minimum wins."""
    d = a.ndim
    if d == 1:
        return 0
    size = math.prod(a.shape)
    best, best_p = math.inf, 0
    for pivot in range(d):
        fibers = len({tuple(np.delete(c, pivot)) for c in a.coords})
        rt, r = [], []
        for k in range(1, d):
            left = math.prod(a.shape[:k])
            bound = min(fibers, left if k <= pivot else size // left)
            rt.append(bound)
            feas = min(bound, left, size // left)
            if target is not None:
                feas = min(feas, target[k - 1])
            r.append(feas)
        cost = modeled_cost(a.shape, pivot, rt, r)
        if cost < best:
            best, best_p = cost, pivot
    return best_p


def lossless_bond_ranks(s: ft.StructuredTT):
    """Interior ranks of the deparallelised exact train (fasttt.py
    _lossless_bond_ranks) through the drop-in itself."""
    return ft.parallel_vector_round(s).ranks[1:-1]
