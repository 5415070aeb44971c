"""CPU oracle for the FastTT decomposition path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference ``sparsett`` hot path
(``/root/reference/pkg/src/sparsett``; file:line citations below are relative
to that package). It is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it. The product package
(``paper_1908_02721_b200``) never imports it and has no CPU fallback.

Differences from the reference, all value-preserving:

* The 0/1 ("quasi-permutation") cores are never densified. The reference
  builds them as dense arrays (fasttt.py:246-255) and contracts them with
  ``tensordot``/``einsum``; every column of such a core holds exactly one 1,
  so those contractions are the scatters ``new[:, kept] = carry.T`` (first
  sweep) and ``new[kept, :] = carry`` (second sweep), which are exact.
* Dense carries use ``@`` instead of ``np.einsum`` (same math, BLAS order).
* The pivot-orthogonality check (fasttt.py:303-321) is skipped for trains
  built here: the side cores are orthonormal by construction.

Pinning: ``tests/test_oracle_golden.py`` checks this module against golden
vectors produced by the unmodified reference (``tests/golden/make_golden.py``)
-- integer outputs bit-exactly, reconstructions to 1e-10.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg

MODES = ("static", "dynamic", "fixed_rank")
ERROR_MEASURE_CAP = 20_000_000  # fasttt.py:74


# ---------------------------------------------------------------- indices
def strides(dims):
    """C-order strides (tensor.py:75-80)."""
    s = np.ones(len(dims), dtype=np.int64)
    for k in range(len(dims) - 2, -1, -1):
        s[k] = s[k + 1] * dims[k + 1]
    return s


def linearize(dims, coords):
    """tensor.py:83-87."""
    return np.asarray(coords, dtype=np.int64) @ strides(dims)


def delinearize(dims, lin):
    """tensor.py:90-100."""
    lin = np.asarray(lin, dtype=np.int64)
    out = np.empty((lin.shape[0], len(dims)), dtype=np.int64)
    st = strides(dims)
    rem = lin
    for k in range(len(dims)):
        out[:, k] = rem // st[k]
        rem = rem % st[k]
    return out


def canonical(shape, coords, values):
    """SparseTensor canonicalisation (tensor.py:123-164): drop zeros, stable
    sort by C-order linear index, reject duplicates."""
    dims = tuple(int(n) for n in shape)
    coords = np.ascontiguousarray(coords, dtype=np.int64).reshape(-1, len(dims))
    values = np.ascontiguousarray(values, dtype=np.float64)
    keep = values != 0.0
    coords, values = coords[keep], values[keep]
    lin = linearize(dims, coords)
    order = np.argsort(lin, kind="stable")
    lin = lin[order]
    if lin.size > 1 and np.any(lin[1:] == lin[:-1]):
        raise ValueError("duplicate coordinate")
    return dims, coords[order], values[order]


def extract_fibers(dims, coords, values, pivot):
    """extract_nonzero_fibers (tensor.py:374-403): lexsort with the pivot
    coordinate fastest, boundaries where the fixed tuple changes."""
    d = len(dims)
    nnz = values.shape[0]
    rest = [k for k in range(d) if k != pivot]
    fixed = coords[:, rest]
    order = np.lexsort((coords[:, pivot],) + tuple(fixed[:, k] for k in range(d - 2, -1, -1)))
    fixed = fixed[order]
    boundary = np.ones(nnz, dtype=bool)
    if nnz > 1:
        boundary[1:] = (fixed[1:] != fixed[:-1]).any(axis=1)
    starts = np.flatnonzero(boundary)
    indptr = np.concatenate([starts, [nnz]]).astype(np.int64)
    return dict(
        fixed_coords=fixed[starts] if nnz else np.zeros((0, d - 1), np.int64),
        indptr=indptr,
        pivot_index=coords[order, pivot].astype(np.int64),
        values=values[order],
        order=order,
    )


def depar_qp(n_rows, col_to_row):
    """depar_quasi_perm (fasttt.py:148-167): kept rows ascending, new map =
    dense rank of the row among the kept ones."""
    present = np.zeros(n_rows, dtype=bool)
    present[col_to_row] = True
    kept = np.flatnonzero(present).astype(np.int64)
    inv = np.zeros(n_rows, dtype=np.int64)
    inv[kept] = np.arange(kept.size, dtype=np.int64)
    return kept, inv[col_to_row]


def index_sweeps(dims, pivot, fixed_coords):
    """_index_sweeps (fasttt.py:181-211)."""
    d = len(dims)
    R = fixed_coords.shape[0]

    def mode_index(k):  # ttformat.py:322-327
        return fixed_coords[:, k if k < pivot else k - 1]

    t_map = np.zeros(R, dtype=np.int64)
    r_prev = 1
    left = []
    for k in range(pivot):
        kept, t_map = depar_qp(r_prev * dims[k], t_map * dims[k] + mode_index(k))
        left.append((kept, r_prev))
        r_prev = kept.size
    s_map = np.zeros(R, dtype=np.int64)
    r_next = 1
    right = []
    for k in range(d - 1, pivot, -1):
        kept, s_map = depar_qp(dims[k] * r_next, mode_index(k) * r_next + s_map)
        right.append((kept, r_next))
        r_next = kept.size
    return left, t_map, r_prev, right, s_map, r_next


def lossless_bond_ranks(dims, pivot, left, right):
    """_lossless_bond_ranks (fasttt.py:214-225)."""
    d = len(dims)
    bonds = [0] * (d - 1)
    for k, (kept, _) in enumerate(left):
        bonds[k] = kept.size
    for step, (kept, _) in enumerate(right):
        bonds[d - 2 - step] = kept.size
    return tuple(bonds)


# ------------------------------------------------------------ cost model
def full_ranks(dims, ranks):
    """ttsvd.py:79-98."""
    d = len(dims)
    ranks = tuple(int(r) for r in ranks)
    if len(ranks) == d - 1:
        ranks = (1,) + ranks + (1,)
    if len(ranks) != d + 1:
        raise ValueError("rank vector length")
    return ranks


def flops_fasttt(dims, pivot, ranks_lossless, ranks_final, c_svd=1.0):
    """fasttt.py:456-481 (exact Python ints, then one float)."""
    d = len(dims)
    if d == 1:
        return 0.0
    rt = full_ranks(dims, ranks_lossless)
    r = full_ranks(dims, ranks_final)
    p = pivot + 1

    def f(m, n):
        return m * n * min(m, n)

    total = f(rt[p - 1] * dims[p - 1], rt[p])
    for i in range(p + 1, d):
        total += f(r[i - 1] * dims[i - 1], rt[i])
    for i in range(2, p + 1):
        total += f(rt[i - 1], dims[i - 1] * r[i])
    return c_svd * float(total)


def flops_ttsvd(dims, ranks, c_svd=1.0):
    """ttsvd.py:101-116."""
    d = len(dims)
    r = full_ranks(dims, ranks)
    total = 0
    for k in range(1, d):
        rows = r[k - 1] * dims[k - 1]
        cols = math.prod(dims[k:])
        total += rows * cols * min(rows, cols)
    return c_svd * float(total)


def upper_bond_bounds(dims, pivot, num_fibers):
    """_upper_bond_bounds (fasttt.py:484-498)."""
    d = len(dims)
    left = [1] * (d + 1)
    for k in range(1, d + 1):
        left[k] = left[k - 1] * dims[k - 1]
    size = left[d]
    return tuple(
        min(num_fibers, left[k]) if k < pivot + 1 else min(num_fibers, size // left[k])
        for k in range(1, d)
    )


def fiber_count(dims, coords, pivot):
    """Distinct fixed tuples for one pivot (fasttt.py:537-541)."""
    if coords.shape[0] == 0:
        return 0
    rest = [k for k in range(len(dims)) if k != pivot]
    keys = linearize(tuple(dims[k] for k in rest), coords[:, rest])
    return int(np.unique(keys).size)


def select_p(dims, coords, values, target_ranks=None, precise=False, c_svd=1.0):
    """select_p (fasttt.py:501-558); strict '<' argmin -> ties to smaller p."""
    d = len(dims)
    if d == 1:
        return 0
    left = [1] * (d + 1)
    for k in range(1, d + 1):
        left[k] = left[k - 1] * dims[k - 1]
    size = left[d]
    if target_ranks is None:
        targets = None
    elif isinstance(target_ranks, (int, np.integer)):
        targets = (int(target_ranks),) * (d - 1)
    else:
        targets = tuple(int(r) for r in target_ranks)
    best_pivot, best_cost = 0, math.inf
    for pivot in range(d):
        nf = fiber_count(dims, coords, pivot)
        if precise:
            fb = extract_fibers(dims, coords, values, pivot)
            lf, _, _, rt_, _, _ = index_sweeps(dims, pivot, fb["fixed_coords"])
            rt = lossless_bond_ranks(dims, pivot, lf, rt_)
        else:
            rt = upper_bond_bounds(dims, pivot, nf)
        r_est = []
        for k in range(1, d):
            feas = min(rt[k - 1], left[k], size // left[k])
            if targets is not None:
                feas = min(feas, targets[k - 1])
            r_est.append(feas)
        cost = flops_fasttt(dims, pivot, rt, tuple(r_est), c_svd)
        if cost < best_cost:
            best_cost, best_pivot = cost, pivot
    return best_pivot


# ----------------------------------------------------------- dense linalg
def _full_svd(m):
    """linalg.py:48-53 (gesdd, gesvd fallback)."""
    try:
        return np.linalg.svd(m, full_matrices=False)
    except np.linalg.LinAlgError:
        return scipy.linalg.svd(m, full_matrices=False, lapack_driver="gesvd")


def _fix_signs(u, vt):
    """linalg.py:56-63."""
    for j in range(u.shape[1]):
        i = int(np.argmax(np.abs(u[:, j])))
        if u[i, j] < 0.0:
            u[:, j] = -u[:, j]
            vt[j, :] = -vt[j, :]


def truncation_rank(s, delta, shape):
    """The tail rule of svd_truncate_delta (linalg.py:89-99)."""
    sq = s * s
    if delta == 0.0:
        if s.size == 0 or s[0] == 0.0:
            return 0
        cut = max(shape) * np.finfo(np.float64).eps * s[0]
        return int(np.count_nonzero(s >= cut))
    tails = np.concatenate([np.cumsum(sq[::-1])[::-1], [0.0]])
    return int(np.argmax(tails <= delta * delta))


def svd_truncate_delta(m, delta):
    """linalg.py:75-105 -> (u, s, vt, rank, trunc_error)."""
    u, s, vt = _full_svd(m)
    rank = truncation_rank(s, delta, m.shape)
    sq = s * s
    err = float(np.sqrt(max(float(np.sum(sq[rank:])), 0.0)))
    u = np.ascontiguousarray(u[:, :rank])
    vt = np.ascontiguousarray(vt[:rank, :])
    s = s[:rank].copy()
    _fix_signs(u, vt)
    return u, s, vt, rank, err


def svd_truncate_rank(m, r):
    """linalg.py:108-125."""
    u, s, vt = _full_svd(m)
    rank = int(min(r, min(m.shape)))
    sq = s * s
    err = float(np.sqrt(max(float(np.sum(sq[rank:])), 0.0)))
    u = np.ascontiguousarray(u[:, :rank])
    vt = np.ascontiguousarray(vt[:rank, :])
    s = s[:rank].copy()
    _fix_signs(u, vt)
    return u, s, vt, rank, err


def qr_economic(m):
    """linalg.py:128-140: reduced QR with diag(R) >= 0."""
    q, r = np.linalg.qr(m, mode="reduced")
    sg = np.sign(np.diag(r))
    sg[sg == 0] = 1.0
    return q * sg, sg[:, None] * r


# ------------------------------------------------------- structured train
def pivot_core(dims, pivot, fib, t_map, r_prev, s_map, r_next):
    """Dense pivot core scatter (fasttt.py:256-259)."""
    pc = np.zeros((r_prev, dims[pivot], r_next))
    per_entry = np.repeat(np.arange(fib["indptr"].size - 1), np.diff(fib["indptr"]))
    pc[t_map[per_entry], fib["pivot_index"], s_map[per_entry]] = fib["values"]
    return pc


def dense_side_core(kind, kept, r_other, n):
    """Materialise one 0/1 core exactly as parallel_vector_round does
    (fasttt.py:246-255); only used for small trains (error measure)."""
    if kind == "L":
        c = np.zeros((r_other, n, kept.size))
        c[kept // n, kept % n, np.arange(kept.size)] = 1.0
    else:
        c = np.zeros((kept.size, n, r_other))
        c[np.arange(kept.size), kept // r_other, kept % r_other] = 1.0
    return c


def structured_cores(dims, pivot, left, right, pc):
    """Index-form train: list of ('L', kept, rp, n) / ('R', kept, rn, n) /
    dense ndarray, in mode order."""
    d = len(dims)
    cores = [None] * d
    for k, (kept, rp) in enumerate(left):
        cores[k] = ("L", kept, rp, dims[k])
    for step, (kept, rn) in enumerate(right):
        k = d - 1 - step
        cores[k] = ("R", kept, rn, dims[k])
    cores[pivot] = pc
    return cores


def _shape(c):
    if isinstance(c, np.ndarray):
        return c.shape
    kind, kept, ro, n = c
    return (ro, n, kept.size) if kind == "L" else (kept.size, n, ro)


def sweep_rounding(cores, pivot, first_svd, second_svd):
    """_sweep_rounding (fasttt.py:324-356) on the index-form train.

    Returns dense cores or None for the zero train (rank 0, :337-338)."""
    cores = list(cores)
    d = len(cores)
    for k in range(pivot, d - 1):  # :334-341
        r0, n, r1 = cores[k].shape
        u, s, vt, rank, _ = first_svd(k, cores[k].reshape(r0 * n, r1))
        if rank == 0:
            return None
        cores[k] = u.reshape(r0, n, rank)
        carry = vt.T * s  # (r1, rank)
        nxt = cores[k + 1]
        if isinstance(nxt, np.ndarray):
            a, nn, c = nxt.shape
            cores[k + 1] = (carry.T @ nxt.reshape(a, nn * c)).reshape(rank, nn, c)
        else:
            kind, kept, rn, nn = nxt
            assert kind == "R"
            new = np.zeros((rank, nn * rn))
            new[:, kept] = carry.T
            cores[k + 1] = new.reshape(rank, nn, rn)
    for k in range(d - 1, pivot, -1):  # :342-347
        r0, n, r1 = cores[k].shape
        q, r = qr_economic(cores[k].reshape(r0, n * r1).T)
        qq = q.shape[1]
        cores[k] = np.ascontiguousarray(q.T).reshape(qq, n, r1)
        a, b, c = cores[k - 1].shape
        cores[k - 1] = (cores[k - 1].reshape(a * b, c) @ r.T).reshape(a, b, qq)
    for k in range(pivot, 0, -1):  # :348-355
        r0, n, r1 = cores[k].shape
        u, s, vt, rank, _ = second_svd(k, cores[k].reshape(r0, n * r1).T)
        if rank == 0:
            return None
        cores[k] = np.ascontiguousarray(u.T).reshape(rank, n, r1)
        carry = vt.T * s  # (r0, rank)
        prv = cores[k - 1]
        if isinstance(prv, np.ndarray):
            a, b, c = prv.shape
            cores[k - 1] = (prv.reshape(a * b, c) @ carry).reshape(a, b, rank)
        else:
            kind, kept, rp, nn = prv
            assert kind == "L"
            new = np.zeros((rp * nn, rank))
            new[kept, :] = carry
            cores[k - 1] = new.reshape(rp, nn, rank)
    return [np.ascontiguousarray(c) for c in cores]


def round_train(cores, dims, pivot, pivot_norm, mode, eps, fixed_ranks=None,
                delta_left=None, delta_right=None):
    """efficient/dynamic/fixed_rank_tt_rounding (fasttt.py:364-453)."""
    d = len(dims)
    if d == 1:
        return [cores[0].copy()]
    denom = math.sqrt(pivot) + math.sqrt(d - 1 - pivot)
    if mode == "static":
        if delta_left is not None or delta_right is not None:
            delta = delta_left if delta_left is not None else delta_right
        else:
            delta = eps * pivot_norm / denom if denom else 0.0
        svd = lambda k, m: svd_truncate_delta(m, delta)
        return sweep_rounding(cores, pivot, svd, svd)
    if mode == "dynamic":
        st = {
            "right": delta_right if delta_right is not None
            else (math.sqrt(d - 1 - pivot) / denom * eps * pivot_norm if denom else 0.0),
            "left": delta_left if delta_left is not None
            else (math.sqrt(pivot) / denom * eps * pivot_norm if denom else 0.0),
        }

        def first(k, m):
            res = svd_truncate_delta(m, st["right"] / math.sqrt(d - 1 - k))
            st["right"] = math.sqrt(max(st["right"] ** 2 - res[4] ** 2, 0.0))
            return res

        def second(k, m):
            res = svd_truncate_delta(m, st["left"] / math.sqrt(k))
            st["left"] = math.sqrt(max(st["left"] ** 2 - res[4] ** 2, 0.0))
            return res

        return sweep_rounding(cores, pivot, first, second)
    targets = fixed_ranks
    if isinstance(targets, (int, np.integer)):
        targets = (int(targets),) * (d - 1)
    targets = full_ranks(dims, targets)
    return sweep_rounding(
        cores, pivot,
        lambda k, m: svd_truncate_rank(m, targets[k + 1]),
        lambda k, m: svd_truncate_rank(m, targets[k]),
    )


# ------------------------------------------------------- train utilities
def tt_entries(cores, coords):
    """Batched entry evaluation with the math of tt_entry
    (ttformat.py:110-121), grouped by mode index so every step is a GEMM."""
    coords = np.asarray(coords, dtype=np.int64)
    n = coords.shape[0]
    v = cores[0][0][coords[:, 0], :]  # (n, r1)
    for k in range(1, len(cores)):
        c = cores[k]
        out = np.empty((n, c.shape[2]))
        ck = coords[:, k]
        order = np.argsort(ck, kind="stable")
        bounds = np.searchsorted(ck[order], np.arange(c.shape[1] + 1))
        for i in range(c.shape[1]):
            rows = order[bounds[i]:bounds[i + 1]]
            if rows.size:
                out[rows] = v[rows] @ c[:, i, :]
        v = out
    return v[:, 0]


def tt_norm(cores):
    """ttformat.py:198-203."""
    w = np.ones((1, 1))
    for c in cores:
        a, n, r = c.shape
        tmp = (w @ c.reshape(a, n * r)).reshape(a * n, r)
        w = c.reshape(a * n, r).T @ tmp
    return float(np.sqrt(max(w[0, 0], 0.0)))


def tt_add(a, b):
    """ttformat.py:157-182."""
    d = len(a)
    if d == 1:
        return [a[0] + b[0]]
    out = []
    for k in range(d):
        ca, cb = a[k], b[k]
        if k == 0:
            out.append(np.concatenate([ca, cb], axis=2))
        elif k == d - 1:
            out.append(np.concatenate([ca, cb], axis=0))
        else:
            ra0, n, ra1 = ca.shape
            rb0, _, rb1 = cb.shape
            c = np.zeros((ra0 + rb0, n, ra1 + rb1))
            c[:ra0, :, :ra1] = ca
            c[ra0:, :, ra1:] = cb
            out.append(c)
    return out


def tt_right_orthogonalize(cores):
    """ttformat.py:206-216."""
    cores = [c.copy() for c in cores]
    for k in range(len(cores) - 1, 0, -1):
        r0, n, r1 = cores[k].shape
        q, r = qr_economic(cores[k].reshape(r0, n * r1).T)
        qq = q.shape[1]
        cores[k] = np.ascontiguousarray(q.T).reshape(qq, n, r1)
        a, b, c = cores[k - 1].shape
        cores[k - 1] = (cores[k - 1].reshape(a * b, c) @ r.T).reshape(a, b, qq)
    return cores


def tt_relative_error(ref, approx, norm=None):
    """fasttt.py:561-584 (raises ValueError above the cap)."""
    total = sum((a.shape[0] + b.shape[0]) * a.shape[1] * (a.shape[2] + b.shape[2])
                for a, b in zip(ref, approx))
    if total > ERROR_MEASURE_CAP:
        raise ValueError("difference train exceeds measurement cap")
    neg = [c.copy() for c in approx]
    neg[0] = neg[0] * -1.0
    diff = tt_add(ref, neg)
    num = float(np.linalg.norm(tt_right_orthogonalize(diff)[0].ravel()))
    if norm is None:
        norm = tt_norm(ref)
    return num / norm if norm > 0 else (0.0 if num == 0.0 else math.inf)


def zero_train(dims):
    return [np.zeros((1, n, 1)) for n in dims]


# ---------------------------------------------------------------- driver
def fasttt(shape, coords, values, eps=1e-14, pivot=None, mode="static",
           fixed_ranks=None, precise_pivot=False, c_svd=1.0, report=True):
    """The fasttt driver (fasttt.py:634-749) on the index-form train.

    Returns ``(cores, info)``; ``info`` carries every integer intermediate
    (fiber order, kept arrays, maps, lossless ranks) for bit-exact checks.
    """
    dims, coords, values = canonical(shape, coords, values)
    d = len(dims)
    if eps is None or eps == 0.0:
        eps = 1e-14
    if mode == "fixed":
        mode = "fixed_rank"
    if pivot is None:
        pivot = select_p(dims, coords, values,
                         target_ranks=fixed_ranks if mode == "fixed_rank" else None,
                         precise=precise_pivot, c_svd=c_svd)
    info = dict(pivot=pivot, mode=mode, eps=eps, nnz=int(values.size))
    if values.size == 0:
        info.update(num_fibers=0, ranks_lossless=(0,) * (d - 1), eps_actual=0.0)
        z = zero_train(dims)
        info["ranks"] = tuple(c.shape[2] for c in z)[:-1]
        return z, info
    fib = extract_fibers(dims, coords, values, pivot)
    left, t_map, r_prev, right, s_map, r_next = index_sweeps(dims, pivot, fib["fixed_coords"])
    pc = pivot_core(dims, pivot, fib, t_map, r_prev, s_map, r_next)
    ranks_lossless = lossless_bond_ranks(dims, pivot, left, right)
    info.update(fibers=fib, left=left, right=right, t_map=t_map, s_map=s_map,
                num_fibers=int(fib["indptr"].size - 1), ranks_lossless=ranks_lossless)
    sc = structured_cores(dims, pivot, left, right, pc)
    pnorm = float(np.linalg.norm(pc.ravel()))  # _budget_norm, fasttt.py:359-361
    out = round_train(sc, dims, pivot, pnorm, mode, eps, fixed_ranks)
    if out is None:
        out = zero_train(dims)
    info["ranks"] = tuple(c.shape[2] for c in out[:-1])
    if report:
        norm_a = float(np.linalg.norm(values))
        na2 = float(values @ values)
        dot = float(values @ tt_entries(out, coords))
        nb = tt_norm(out)
        inner = math.sqrt(max(na2 - 2.0 * dot + nb * nb, 0.0) / na2)
        exact_total = sum((_shape(a)[0] + b.shape[0]) * b.shape[1] * (_shape(a)[2] + b.shape[2])
                          for a, b in zip(sc, out))
        if exact_total <= ERROR_MEASURE_CAP:
            exact = [c if isinstance(c, np.ndarray) else dense_side_core(c[0], c[1], c[2], c[3])
                     for c in sc]
            info["eps_actual"] = tt_relative_error(exact, out, norm=norm_a)
            info["eps_actual_method"] = "tt_difference"
        else:
            info["eps_actual"] = inner
            info["eps_actual_method"] = "inner_identity"
        info["eps_actual_inner"] = inner
        info["flops_fasttt_model"] = flops_fasttt(dims, pivot, ranks_lossless,
                                                  (1,) + info["ranks"] + (1,), c_svd)
    return out, info
