"""GPU parity against the UNMODIFIED reference (and, where the reference
cannot run, the pinned oracle) on every BASELINE config -- the north-star
bar: integer outputs bit-exact; reconstructed entries within 1e-10 relative
Frobenius error over every nonzero plus 1e6 seeded zero positions
(``G.zero_positions(shape, coords, 1_000_000, seed=99)``).

Fixtures come from tests/golden/make_golden.py (targets c{N}_z1m, c5train,
refmid, fdm, tensorize, acceptance).  Reference trains are evaluated by the
test-side torch evaluator (tests/tteval.py), the GPU trains by the product's
``tt_entries``.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from tteval import tt_entries_torch
import paper_1908_02721_b200 as ft
from paper_1908_02721_b200 import generators as G

pytestmark = pytest.mark.gpu

RECON_TOL = 1e-10
Z1M, Z1M_SEED = 1_000_000, 99


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def rel_err(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _meta(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        return json.load(fh)


def _z1m(t, meta_digest):
    zc = G.zero_positions(t.shape, t.coords, Z1M, seed=Z1M_SEED)
    assert digest(zc) == meta_digest
    return zc


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_config_entries_nnz_and_1e6_zeros(cfg):
    """The decomposition at the reference's auto pivot against the golden
    train (c1: the reference's own fasttt; c2/c4: the oracle, the reference
    raises MemoryError there; c3: the oracle) at every nonzero and 1e6
    seeded zero positions."""
    meta, z = load_golden(f"c{cfg}")
    zm = _meta(f"c{cfg}_z1m")
    ref_z = np.load(os.path.join(GOLDEN, f"c{cfg}_z1m.npz"))["entries"]
    shape, coords, vals, eps = G.gen_config(cfg)
    t = ft.SparseTensor(shape, coords, vals)
    tt, rep = ft.fasttt(t, eps=eps)
    assert rep.pivot == meta["auto_pivot"]
    assert list(rep.ranks) == meta["ranks"] == zm["ranks"]
    zc = _z1m(t, zm["coords"])
    got = np.concatenate([ft.tt_entries(tt, t.coords), ft.tt_entries(tt, zc)])
    want = np.concatenate([z["entries_nnz"], ref_z])
    assert rel_err(got, want) <= RECON_TOL


@pytest.mark.slow
def test_config5_against_oracle_train():
    """Config 5 at the auto pivot p = 2 against the oracle's train (LAPACK
    gesdd on the 4160 x 314,928 dense pivot core; the reference itself would
    allocate a 314,928 x 32 x 104,976 core): ranks, entries at all 8.5M
    nonzeros and at 1e6 seeded zero positions."""
    m = _meta("c5train")
    zref = np.load(os.path.join(GOLDEN, "c5train.npz"))
    cores = [zref[f"core{k}"] for k in range(12)]
    shape, coords, vals, eps = G.gen_config(5)
    t = ft.SparseTensor(shape, coords, vals)
    tt, rep = ft.fasttt(t, eps=eps)
    assert rep.pivot == m["pivot"]
    assert list(rep.ranks_lossless) == m["ranks_lossless"]
    assert list(rep.ranks) == m["ranks"]
    zc = _z1m(t, m["z1m_coords"])
    got = np.concatenate([ft.tt_entries(tt, t.coords), ft.tt_entries(tt, zc)])
    want = np.concatenate([tt_entries_torch(cores, t.coords), zref["entries_z1m"]])
    assert rel_err(got, want) <= RECON_TOL
    # the checker itself agrees with the oracle's committed evaluation
    assert rel_err(tt_entries_torch(cores, zc[:1000]), zref["entries_z1m"][:1000]) <= 1e-12 or \
        np.abs(tt_entries_torch(cores, zc[:1000]) - zref["entries_z1m"][:1000]).max() <= 1e-15


@pytest.mark.parametrize("cfg,pivot", [(2, 2), (4, 3)])
def test_reference_train_at_middle_pivot(cfg, pivot):
    """The unmodified reference's own fasttt(t, eps, pivot) where it fits in
    memory (c2 at p = 2, c4 at p = 3): integer report fields bit-exact, the
    flop models exactly, entries at every nonzero and 1e6 zero positions."""
    m = _meta(f"c{cfg}_ref_p{pivot}")
    z = np.load(os.path.join(GOLDEN, f"c{cfg}_ref_p{pivot}.npz"))
    shape, coords, vals, eps = G.gen_config(cfg)
    t = ft.SparseTensor(shape, coords, vals)
    tt, rep = ft.fasttt(t, eps=eps, pivot=pivot)
    assert rep.num_fibers == m["num_fibers"]
    assert list(rep.ranks_lossless) == m["ranks_lossless"]
    assert list(rep.ranks) == m["ranks"]
    assert rep.flops_fasttt_model == m["flops_fasttt_model"]
    assert rep.flops_ttsvd_model == m["flops_ttsvd_model"]
    assert rep.eps_actual_method == m["eps_actual_method"]
    # the inner-product identity resolves ~1e-8 (the reference clamps its
    # negative rounding noise to 0, fasttt.py:561-602): equal within 1e-6,
    # the reference acceptance gate's floor; the TT difference within 1e-9
    tol = 1e-6 if m["eps_actual_method"] == "inner_identity" else 1e-9
    assert abs(rep.eps_actual - m["eps_actual"]) <= tol
    zc = _z1m(t, m["z1m_coords"])
    got = np.concatenate([ft.tt_entries(tt, t.coords), ft.tt_entries(tt, zc)])
    want = np.concatenate([z["entries_nnz"], z["entries_z1m"]])
    assert rel_err(got, want) <= RECON_TOL
    if m["cores_stored"]:
        ref = [z[f"core{k}"] for k in range(t.ndim)]
        assert rel_err(tt_entries_torch(ref, t.coords), z["entries_nnz"]) <= 1e-14


def test_config4_input_through_reference_tensorize():
    """Config 4's tensor equals the reference's tensorize_matrix
    (ttformat.py:414-433) of the same D L D matrix, bit for bit, through the
    drop-in's host and device tensorize_matrix and the bench generator."""
    import scipy.sparse as sp

    m = _meta("c4_tensorize")
    rows, cols, v, n = G.laplacian_2d_scaled(256, np.random.default_rng(0))
    assert (digest(rows), digest(cols), digest(v)) == (m["matrix_rows"], m["matrix_cols"],
                                                      m["matrix_values"])
    mat = sp.coo_matrix((v, (rows, cols)), shape=(n, n))
    dims = tuple(m["row_dims"])
    for t in (ft.tensorize_matrix(mat, dims, dims), ft.tensorize_matrix(mat, dims, dims, device=True),
              ft.SparseTensor(*G.gen_config(4)[:3])):
        assert list(t.shape) == m["shape"] and t.nnz == m["nnz"]
        assert digest(t.coords) == m["coords"]
        assert digest(t.values) == m["values"]


@pytest.mark.parametrize("case", ["lap", "rnd"])
@pytest.mark.parametrize("device", [False, True])
def test_fdm_mpo_known_answers(case, device):
    """The paper's MPO experiment as the reference's acceptance gate runs it
    (test_acceptance.py:87-107, 207-228): 20^3 7-point stencil matrices from
    the reference's gen_fdm (committed), tensorized (20,20,20) x (20,20,20),
    fasttt(eps=1e-14, pivot=1): R = 1920, r~ = (58, 58), ranks (2, 2) for the
    Laplacian (eps_actual <= 1e-12) and (58, 58) for the seed-1234 random
    coefficients (eps_actual <= 5e-14); entries against the reference's train
    at every nonzero and 1e6 seeded zero positions."""
    import scipy.sparse as sp

    meta = _meta("fdm")
    z = np.load(os.path.join(GOLDEN, "fdm.npz"))
    ref = meta[case]
    mat = sp.coo_matrix((z[f"{case}_val"], (z[f"{case}_row"].astype(np.int64),
                                            z[f"{case}_col"].astype(np.int64))),
                        shape=tuple(ref["shape"]))
    dims = tuple(meta["dims"])
    t = ft.tensorize_matrix(mat, dims, dims, device=device)
    assert digest(t.coords) == ref["coords"] and digest(t.values) == ref["values"]
    tt, rep = ft.fasttt(t, eps=meta["eps"], pivot=meta["pivot"])
    assert rep.num_fibers == ref["num_fibers"] == 1920
    assert list(rep.ranks_lossless) == ref["ranks_lossless"] == [58, 58]
    assert list(rep.ranks) == ref["ranks"]
    assert rep.eps_actual <= (1e-12 if case == "lap" else 5e-14)
    cores = [z[f"{case}_core{k}"] for k in range(3)]
    zc = G.zero_positions(t.shape, t.coords, Z1M, seed=Z1M_SEED)
    pts = np.concatenate([t.coords, zc])
    assert rel_err(ft.tt_entries(tt, pts), tt_entries_torch(cores, pts)) <= RECON_TOL
    mpo = ft.tt_split_mpo(tt, dims, dims)
    assert [c.shape[1:3] for c in mpo.cores] == [(20, 20)] * 3


# ------------------------------------------------------------ acceptance gate
def _suite():
    meta = _meta("acceptance")
    z = np.load(os.path.join(GOLDEN, "acceptance.npz"))
    off = z["suite_off"]
    out = []
    for i, case in enumerate(meta["cases"]):
        shape = tuple(case["shape"])
        lin = z["suite_lin"][off[i]:off[i + 1]].astype(np.int64)
        coords = np.stack(np.unravel_index(lin, shape), 1).astype(np.int64)
        out.append((ft.SparseTensor(shape, coords, z["suite_val"][off[i]:off[i + 1]]), case))
    return meta, z, out


def test_acceptance_criteria_1_2_4_lossless():
    """Criteria 1, 2, 4 of the reference's acceptance gate
    (test_acceptance.py:110-204) on its 200-tensor suite, plus bit-exact
    agreement with the reference's own runs: pivot, R, r~ and final ranks of
    every tensor equal the reference's; worst eps_actual <= 1e-11 and inner
    identity <= 1e-6; ranks equal the classical TT-SVD's; r~_k <= min(R,
    outer extent)."""
    meta, _, suite = _suite()
    worst = worst_inner = 0.0
    for t, case in suite:
        tt, rep = ft.fasttt(t, eps=1e-14)
        assert rep.pivot == case["pivot"]
        assert rep.num_fibers == case["num_fibers"]
        assert list(rep.ranks_lossless) == case["ranks_lossless"]
        assert list(rep.ranks) == case["ranks"] == case["ttsvd_ranks"][1:-1]
        assert rep.eps_actual_method == case["eps_actual_method"]
        worst = max(worst, rep.eps_actual)
        worst_inner = max(worst_inner, ft.sparse_inner_error(t, tt))
        left = 1
        for k in range(1, t.ndim):
            left *= t.shape[k - 1]
            outer = left if k <= rep.pivot else t.size // left
            assert rep.ranks_lossless[k - 1] <= min(rep.num_fibers, outer)
    assert worst <= 1e-11 and worst_inner <= 1e-6, (worst, worst_inner)


def test_acceptance_criterion_3_error_bound():
    """Criterion 3 (test_acceptance.py:170-188): 1,200 rounded runs (eps in
    {0.5, 0.1, 0.01} x static/dynamic) with eps_actual <= eps + 1e-12, and
    every run's pivot and ranks equal to the reference's."""
    meta, _, suite = _suite()
    runs = 0
    for t, case in suite:
        for want in case["rounded"]:
            _, rep = ft.fasttt(t, eps=want["eps"], mode=want["mode"])
            runs += 1
            assert rep.eps_actual <= want["eps"] + 1e-12
            assert rep.pivot == want["pivot"]
            assert list(rep.ranks) == want["ranks"], (t.shape, want)
            assert list(rep.ranks_lossless) == want["ranks_lossless"]
    assert runs == 1200


def test_acceptance_criterion_4_quasi_perm():
    """Criterion 4's quasi-permutation half (test_acceptance.py:190-204): the
    reference's rng(4) inputs, depar_quasi_perm's kept rows and map digests
    equal the reference's and beta <= n_rows."""
    meta, z, _ = _suite()
    off = z["qp_off"]
    for i, want in enumerate(meta["qp"]):
        rows = int(z["qp_rows"][i])
        ctr = z["qp_ctr"][off[i]:off[i + 1]].astype(np.int64)
        n, tq = ft.depar_quasi_perm(ft.QuasiPermMatrix(rows, ctr.size, ctr))
        assert n.n_cols == want["n_cols"] <= rows
        assert digest(np.asarray(n.col_to_row)) == want["kept"]
        assert digest(np.asarray(tq.col_to_row)) == want["t_map"]


def test_acceptance_criterion_8_pivot_selection():
    """Criterion 8 (test_acceptance.py:267-277): the image-shape tensor from
    the reference's gen_random_sparse(seed 42, fill_last_mode) with target
    rank 100 selects mode 7 (1-based)."""
    meta, z, _ = _suite()
    c8 = meta["criterion8"]
    shape = tuple(c8["shape"])
    coords = np.stack(np.unravel_index(z["c8_lin"], shape), 1).astype(np.int64)
    t = ft.SparseTensor(shape, coords, z["c8_val"])
    assert t.nnz == c8["nnz"]
    assert ft.select_p(t, target_ranks=100) == c8["select_p_target100"] == 6


def test_tt_entries_negative_and_out_of_range_indices():
    """tt_entries keeps the reference's numpy indexing contract on the GPU
    path: negative indices wrap, out-of-range ones raise IndexError before
    any kernel reads a core."""
    rng = np.random.default_rng(5)
    dims = (4, 6, 5)
    cores = [rng.standard_normal((1 if k == 0 else 3, n, 1 if k == 2 else 3))
             for k, n in enumerate(dims)]
    tt = ft.TTTensor(cores)
    pos = np.stack([rng.integers(0, n, 500) for n in dims], 1)
    neg = pos - np.asarray(dims)
    assert np.array_equal(ft.tt_entries(tt, neg), ft.tt_entries(tt, pos))
    with pytest.raises(IndexError, match="out of bounds for axis 1 with size 6"):
        ft.tt_entries(tt, np.array([[0, 6, 0]]))


def test_contexts_are_per_thread():
    """Two threads decomposing at once (each gets its own native context:
    arena and SVD state) give the same trains as one thread alone."""
    import threading

    shape, coords, vals, eps = G.gen_config(2)
    t = ft.SparseTensor(shape, coords, vals)
    ref_tt, ref_rep = ft.fasttt(t, eps=eps)
    want = ft.tt_entries(ref_tt, t.coords[:5000])
    out = {}

    def run(i):
        import torch

        with torch.cuda.stream(torch.cuda.Stream()):
            tt, rep = ft.fasttt(t, eps=eps)
            torch.cuda.current_stream().synchronize()
        out[i] = (rep.ranks, ft.tt_entries(tt, t.coords[:5000]))

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for i in range(2):
        assert out[i][0] == ref_rep.ranks
        assert rel_err(out[i][1], want) <= 1e-12
