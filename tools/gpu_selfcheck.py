"""Kernel-by-kernel self check on a GPU box (debug aid; prints PASS/FAIL per
check and keeps going). Uses the oracle as the checker only."""

from __future__ import annotations

import json
import math
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from oracle import fasttt_oracle as O  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402
from paper_1908_02721_b200 import pipeline as P  # noqa: E402
from paper_1908_02721_b200 import trains as T  # noqa: E402

results = []


def check(name):
    def deco(fn):
        t0 = time.time()
        try:
            msg = fn()
            ok = True
        except Exception as e:  # noqa: BLE001
            ok = False
            msg = f"{type(e).__name__}: {e}\n" + traceback.format_exc(limit=4)
        dt = time.time() - t0
        print(f"{'PASS' if ok else 'FAIL'} {name} ({dt:.2f}s) {msg or ''}", flush=True)
        results.append((name, ok))
        return fn
    return deco


def rand_sparse(rng, shape, density):
    size = math.prod(shape)
    nnz = max(1, int(density * size))
    lin = np.sort(rng.permutation(size)[:nnz].astype(np.int64))
    vals = rng.uniform(-1, 1, nnz)
    vals[vals == 0] = 0.5
    return ft.SparseTensor(shape, O.delinearize(shape, lin), vals)


rng = np.random.default_rng(7)
SMALL = [rand_sparse(rng, s, 0.2) for s in [(4, 5, 6), (3, 3, 3, 3), (2, 6, 3, 4), (8, 9),
                                             (5, 4, 6, 3), (6, 5, 4), (2, 2, 2, 2, 2)]]


@check("fiber_counts")
def _():
    for t in SMALL:
        got = P._fiber_counts_device(t)
        want = [O.fiber_count(t.shape, t.coords, p) for p in range(t.ndim)]
        assert got == want, (t.shape, got, want)


@check("extract_fibers")
def _():
    for t in SMALL:
        for p in range(t.ndim):
            fs = ft.extract_nonzero_fibers(t, p)
            ref = O.extract_fibers(t.shape, t.coords, t.values, p)
            assert np.array_equal(fs.indptr, ref["indptr"])
            assert np.array_equal(fs.fixed_coords, ref["fixed_coords"])
            assert np.array_equal(fs.pivot_index, ref["pivot_index"])
            assert np.array_equal(fs.values, ref["values"])


@check("index_sweeps")
def _():
    for t in SMALL:
        for p in range(t.ndim):
            s = ft.build_structured_tt(t, p)
            df = P._device_fibers_of(s)
            sw = P.index_sweeps_device(df)
            ref = O.index_sweeps(t.shape, p, O.extract_fibers(t.shape, t.coords, t.values, p)["fixed_coords"])
            left, t_map, r_prev, right, s_map, r_next = ref
            assert sw.r_prev == r_prev and sw.r_next == r_next
            for (a, ra), (b, rb) in zip(sw.left, left):
                assert np.array_equal(a.cpu().numpy(), b) and ra == rb
            for (a, ra), (b, rb) in zip(sw.right, right):
                assert np.array_equal(a.cpu().numpy(), b) and ra == rb
            if p > 0:
                assert np.array_equal(sw.t_map.cpu().numpy(), t_map)
            if p < t.ndim - 1:
                assert np.array_equal(sw.s_map.cpu().numpy(), s_map)


@check("depar_quasi_perm")
def _():
    r = np.random.default_rng(3)
    for rows, cols in [(9, 14), (7, 30), (40, 200), (1, 5), (5000, 300), (3_000_000, 1000)]:
        q = ft.QuasiPermMatrix(rows, cols, r.integers(0, rows, cols))
        n, tm = ft.depar_quasi_perm(q)
        kept, tmap = O.depar_qp(rows, q.col_to_row)
        assert np.array_equal(n.col_to_row, kept), rows
        assert np.array_equal(tm.col_to_row, tmap), rows


@check("dgemm")
def _():
    r = np.random.default_rng(5)
    worst = 0.0
    for (m, n, k) in [(1, 1, 1), (7, 5, 3), (64, 64, 16), (65, 63, 17), (130, 70, 300),
                      (32, 100, 5000), (3, 2, 100000), (500, 400, 90)]:
        for ta in (0, 1):
            for tb in (0, 1):
                A = r.standard_normal((k, m) if ta else (m, k))
                B = r.standard_normal((n, k) if tb else (k, n))
                C0 = r.standard_normal((m, n))
                # column-major: pass transposed numpy (row-major) buffers
                Ad = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
                Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
                Cd = torch.from_numpy(np.ascontiguousarray(C0.T)).cuda()
                lda = A.shape[0]
                ldb = B.shape[0]
                T.dgemm(ta, tb, m, n, k, 1.5, Ad, lda, Bd, ldb, -0.5, Cd, m)
                want = 1.5 * ((A.T if ta else A) @ (B.T if tb else B)) - 0.5 * C0
                got = Cd.cpu().numpy().T
                err = np.abs(got - want).max() / max(1.0, np.abs(want).max())
                worst = max(worst, err)
                assert err < 1e-12, (m, n, k, ta, tb, err)
    return f"max rel err {worst:.2e}"


@check("qr")
def _():
    r = np.random.default_rng(11)
    worst = 0.0
    for (m, n) in [(1, 1), (5, 3), (3, 5), (40, 40), (100, 37), (300, 129), (129, 300),
                   (2000, 64), (5000, 260), (70000, 40)]:
        A = r.standard_normal((m, n))
        res = ft.qr_economic(A)
        q0, r0 = np.linalg.qr(A)
        sg = np.sign(np.diag(r0)); sg[sg == 0] = 1
        q0, r0 = q0 * sg, sg[:, None] * r0
        e1 = np.abs(res.q @ res.r - A).max()
        e2 = np.abs(res.q.T @ res.q - np.eye(min(m, n))).max()
        e3 = np.abs(res.r - r0).max()
        worst = max(worst, e1, e2, e3)
        assert np.all(np.diag(res.r) >= 0)
        assert e1 < 1e-11 and e2 < 1e-12 and e3 < 1e-10, (m, n, e1, e2, e3)
    return f"worst {worst:.2e}"


@check("svd")
def _():
    r = np.random.default_rng(13)
    worst = 0.0
    for (m, n, rk) in [(1, 1, 1), (6, 4, 4), (4, 6, 4), (30, 20, 20), (100, 37, 5), (37, 100, 5),
                       (300, 300, 300), (500, 64, 8), (4096, 200, 16), (200, 3000, 200),
                       (1000, 700, 300)]:
        A = r.standard_normal((m, rk)) @ r.standard_normal((rk, n))
        A /= np.linalg.norm(A)
        res = ft.svd_truncate_rank(A, min(m, n))
        s0 = np.linalg.svd(A, compute_uv=False)
        e1 = np.abs(res.s - s0).max()
        e2 = np.abs((res.u * res.s) @ res.vt - A).max()
        worst = max(worst, e1, e2)
        assert e1 < 1e-13 and e2 < 1e-12, (m, n, rk, e1, e2)
        d = ft.svd_truncate_delta(A, 1e-10)
        ref = O.svd_truncate_delta(A, 1e-10)
        assert d.rank == ref[3], (m, n, d.rank, ref[3])
        if d.rank:
            assert np.abs(d.u @ np.diag(d.s) @ d.vt - ref[0] @ np.diag(ref[1]) @ ref[2]).max() < 1e-12
    return f"worst {worst:.2e}"


@check("tt_entries")
def _():
    r = np.random.default_rng(17)
    for dims, ranks in [((4, 5, 6), (3, 2)), ((3, 3, 3, 3), (9, 27, 9)), ((5, 7, 4, 6), (70, 100, 80)),
                        ((16, 16, 16), (16, 200))]:
        full = (1,) + ranks + (1,)
        cores = [r.standard_normal((full[k], n, full[k + 1])) for k, n in enumerate(dims)]
        coords = np.stack([r.integers(0, n, 3000) for n in dims], 1)
        got = ft.tt_entries(ft.TTTensor(cores), coords)
        want = O.tt_entries(cores, coords)
        err = np.abs(got - want).max() / np.abs(want).max()
        assert err < 1e-12, (dims, ranks, err)
        nrm = ft.tt_norm(ft.TTTensor(cores))
        assert abs(nrm - O.tt_norm(cores)) / nrm < 1e-12


@check("fasttt_small_vs_oracle")
def _():
    worst = 0.0
    for t in SMALL:
        for p in range(t.ndim):
            for mode, eps, kw in (("static", 1e-14, {}), ("static", 0.1, {}), ("dynamic", 0.1, {}),
                                  ("fixed_rank", None, {"fixed_ranks": 2})):
                tt, rep = ft.fasttt(t, eps=eps, pivot=p, mode=mode, **kw)
                oc, oi = O.fasttt(t.shape, t.coords, t.values, eps=eps, pivot=p, mode=mode, **kw)
                assert tuple(rep.ranks) == oi["ranks"], (t.shape, p, mode, rep.ranks, oi["ranks"])
                assert tuple(rep.ranks_lossless) == oi["ranks_lossless"]
                allc = np.concatenate([t.coords, G.zero_positions(t.shape, t.coords, 50)])
                a = O.tt_entries([np.asarray(c) for c in tt.cores], allc)
                b = O.tt_entries(oc, allc)
                err = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
                worst = max(worst, err)
                assert err < 1e-10, (t.shape, p, mode, err)
                assert abs(rep.eps_actual - oi["eps_actual"]) < 1e-9, (rep.eps_actual, oi["eps_actual"])
    return f"worst rel err {worst:.2e}"


def config_check(cfg):
    shape, coords, vals, eps = G.gen_config(cfg)
    t = ft.SparseTensor(shape, coords, vals)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"c{cfg}.json")))
    z = np.load(os.path.join(ROOT, "tests", "golden", f"c{cfg}.npz"))
    torch.cuda.synchronize()
    t0 = time.time()
    tt, rep = ft.fasttt(t, eps=eps)
    t1 = time.time()
    assert rep.pivot == gold["auto_pivot"], (rep.pivot, gold["auto_pivot"])
    assert list(rep.ranks_lossless) == gold["index"]["ranks_lossless"]
    assert list(rep.ranks) == gold["ranks"], (rep.ranks, gold["ranks"])
    cores = [np.asarray(c) for c in tt.cores]
    a = np.concatenate([O.tt_entries(cores, t.coords), O.tt_entries(cores, z["zero_coords"])])
    b = np.concatenate([z["entries_nnz"], z["entries_zero"]])
    err = np.linalg.norm(a - b) / np.linalg.norm(b)
    assert err < 1e-10, err
    # second run (warm)
    torch.cuda.synchronize()
    t2 = time.time()
    ft.fasttt(t, eps=eps)
    torch.cuda.synchronize()
    t3 = time.time()
    return f"err {err:.2e} first {t1 - t0:.2f}s warm {t3 - t2:.3f}s nnz/s {t.nnz / (t3 - t2):.3e} eps_actual {rep.eps_actual:.2e}"


for cfg in [int(c) for c in os.environ.get("CFGS", "1,2,4").split(",") if c]:
    check(f"config{cfg}")(lambda cfg=cfg: config_check(cfg))

print("SUMMARY", sum(ok for _, ok in results), "/", len(results), flush=True)
