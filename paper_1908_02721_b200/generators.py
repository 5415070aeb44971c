"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference ships no generator for these configurations (its
``generators.py`` only has the 3-D 7-point FDM stencil and a uniform random
tensor), so they are defined here from the BASELINE.json wording. All
randomness comes from ``numpy.random.default_rng(seed)`` (PCG64), drawn in
the fixed order documented on each function, so every input is reproducible
from ``(config, seed)``.

The generators return plain arrays (``shape, coords, values``) with
coincident coordinates already summed (BASELINE.json: "coordinates that
coincide are summed"); wrapping them in a :class:`SparseTensor` sorts them
into the canonical C order.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = [
    "CONFIGS",
    "sum_of_rank1",
    "laplacian_2d_scaled",
    "gen_config",
    "zero_positions",
]


def _coalesce(shape, lin: np.ndarray, vals: np.ndarray):
    """Sum values that share a linear index; drop exact zeros."""
    uniq, inv = np.unique(lin, return_inverse=True)
    summed = np.zeros(uniq.size)
    np.add.at(summed, inv, vals)
    keep = summed != 0.0
    uniq = uniq[keep]
    summed = summed[keep]
    coords = np.empty((uniq.size, len(shape)), dtype=np.int64)
    rem = uniq.copy()
    for k in range(len(shape) - 1, -1, -1):
        coords[:, k] = rem % shape[k]
        rem //= shape[k]
    return coords, summed


def _strides(shape):
    s = [1] * len(shape)
    for k in range(len(shape) - 2, -1, -1):
        s[k] = s[k + 1] * shape[k + 1]
    return np.asarray(s, dtype=np.int64)


def sum_of_rank1(shape, terms: int, support: int, dist: str, rng, extra: int = 0,
                 extra_sigma: float = 0.0):
    """Sum of ``terms`` rank-1 tensors with ``support`` nonzeros per factor.

    Draw order, per term ``r`` then per mode ``k``: ``support`` distinct
    positions (``rng.choice(n_k, support, replace=False)``) then their values
    (``U(0.5, 1.5)`` or ``N(0, 1)``). Then, when ``extra`` > 0, ``extra``
    uniform coordinates (one ``rng.integers`` call per mode) with values
    ``N(0, extra_sigma)`` (sigma read as a standard deviation).
    """
    d = len(shape)
    strides = _strides(shape)
    lins = []
    vals = []
    for _ in range(terms):
        pos = []
        fac = []
        for k in range(d):
            p = rng.choice(shape[k], support, replace=False).astype(np.int64)
            if dist == "uniform":
                v = rng.uniform(0.5, 1.5, support)
            else:
                v = rng.standard_normal(support)
            pos.append(p)
            fac.append(v)
        # outer product of the supports: last mode fastest
        lin = np.zeros(1, dtype=np.int64)
        val = np.ones(1)
        for k in range(d):
            lin = (lin[:, None] + pos[k][None, :] * strides[k]).ravel()
            val = (val[:, None] * fac[k][None, :]).ravel()
        lins.append(lin)
        vals.append(val)
    if extra:
        cols = [rng.integers(0, shape[k], extra, dtype=np.int64) for k in range(d)]
        lin = np.zeros(extra, dtype=np.int64)
        for k in range(d):
            lin += cols[k] * strides[k]
        lins.append(lin)
        vals.append(rng.normal(0.0, extra_sigma, extra))
    return _coalesce(shape, np.concatenate(lins), np.concatenate(vals))


def laplacian_2d_scaled(grid: int, rng):
    """``D L D`` for the 2-D 5-point Laplacian on a ``grid x grid`` mesh.

    ``L = kron(T, I) + kron(I, T)`` with ``T = tridiag(-1, 2, -1)``; ``D`` is
    diagonal with ``U(0.5, 1.5)`` entries (one ``rng.uniform`` call of length
    ``grid**2``). Returns COO ``(rows, cols, vals, n)`` sorted by (row, col).
    """
    n = grid * grid
    dvec = rng.uniform(0.5, 1.5, n)
    idx = np.arange(n, dtype=np.int64)
    gi = idx // grid
    gj = idx % grid
    rows = [idx]
    cols = [idx]
    vals = [np.full(n, 4.0)]
    for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        ok = (gi + di >= 0) & (gi + di < grid) & (gj + dj >= 0) & (gj + dj < grid)
        r = idx[ok]
        c = (gi[ok] + di) * grid + (gj[ok] + dj)
        rows.append(r)
        cols.append(c)
        vals.append(np.full(r.size, -1.0))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals) * dvec[rows] * dvec[cols]
    order = np.lexsort((cols, rows))
    return rows[order], cols[order], vals[order], n


# name, shape, eps, builder
CONFIGS = {
    1: dict(name="c1_100^4_R5_s10", shape=(100,) * 4, eps=1e-10),
    2: dict(name="c2_64^6_R8_s6", shape=(64,) * 6, eps=1e-10),
    3: dict(name="c3_16^10_R4_s3_noise2000", shape=(16,) * 10, eps=1e-8),
    4: dict(name="c4_lap2d_256_DLD_mpo_4x4x8", shape=(16,) * 8, eps=1e-10,
            row_dims=(4,) * 8, col_dims=(4,) * 8),
    5: dict(name="c5_32^12_R16_s3", shape=(32,) * 12, eps=1e-10),
}


def gen_config(cfg: int, seed: int = 0):
    """Return ``(shape, coords, values, eps)`` for BASELINE config ``cfg``.

    Config 4 is the tensorized matrix (16^8 fused modes); the matrix COO is
    available from :func:`laplacian_2d_scaled`.
    """
    rng = np.random.default_rng(seed)
    c = CONFIGS[cfg]
    shape = c["shape"]
    if cfg == 1:
        coords, vals = sum_of_rank1(shape, 5, 10, "uniform", rng)
    elif cfg == 2:
        coords, vals = sum_of_rank1(shape, 8, 6, "normal", rng)
    elif cfg == 3:
        coords, vals = sum_of_rank1(shape, 4, 3, "uniform", rng, extra=2000,
                                    extra_sigma=1e-3)
    elif cfg == 4:
        import scipy.sparse

        from .trains import tensorize_matrix

        rows, cols, v, n = laplacian_2d_scaled(256, rng)
        t = tensorize_matrix(scipy.sparse.coo_matrix((v, (rows, cols)), shape=(n, n)),
                             c["row_dims"], c["col_dims"])
        shape, coords, vals = t.shape, np.array(t.coords), np.array(t.values)
    elif cfg == 5:
        coords, vals = sum_of_rank1(shape, 16, 3, "normal", rng)
    else:
        raise ValueError(f"unknown config {cfg}")
    return tuple(shape), coords, vals, c["eps"]


def zero_positions(shape, coords, count: int, seed: int = 12345):
    """``count`` uniform coordinates that are not stored nonzeros, from a
    separate seeded stream (rejection against the stored linear indices)."""
    rng = np.random.default_rng(seed)
    strides = _strides(shape)
    stored = np.sort(coords.astype(np.int64) @ strides)
    out = []
    have = 0
    total = math.prod(shape)
    while have < count:
        cand = np.stack([rng.integers(0, n, count, dtype=np.int64) for n in shape], 1)
        lin = cand @ strides
        pos = np.searchsorted(stored, lin)
        pos = np.minimum(pos, max(stored.size - 1, 0))
        hit = stored.size > 0
        ok = ~(hit & (stored[pos] == lin)) if stored.size else np.ones(count, bool)
        cand = cand[ok]
        out.append(cand)
        have += cand.shape[0]
        if total <= stored.size:
            break
    return np.concatenate(out)[:count]
