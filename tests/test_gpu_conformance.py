"""Reference conformance: the hot-path contracts of the reference's own unit
tests (pkg/tests/test_fasttt.py, test_linalg.py and the fiber tests of
test_tensor.py) checked against the drop-in on the GPU.

The checks are restated here (the reference tree does not travel to the GPU
box); each group cites the reference test class it follows.  Test-only
helpers the reference imports from ``sparsett`` (tt_to_full, tt_svd,
structured_to_tt, as_quasi_perm, the brute-force pivot model) live in
tests/refshim.py, not in the product.
"""

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1908_02721_b200 as ft
from refshim import (as_quasi_perm, brute_select, lossless_bond_ranks, modeled_cost, rand_sparse,
                     structured_to_tt, tt_svd, tt_to_full)

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


# ---- depar_general (test_fasttt.py TestDeparGeneral) ---------------------

def test_depar_general_planted_classes(rng):
    u, v, w = (rng.standard_normal(6) for _ in range(3))
    m = np.column_stack([u, 2.0 * u, v, np.zeros(6), -3.0 * v, w])
    n, t = ft.depar_general(m)
    assert n.shape == (6, 3)
    for j, ref in enumerate((u, v, w)):
        assert np.array_equal(n[:, j], ref)  # first occurrence kept verbatim
    assert np.allclose(n @ t, m, atol=1e-12)
    assert not np.any(t[:, 3])  # the zero column maps to nothing


def test_depar_general_degenerate_inputs(rng):
    n, t = ft.depar_general(np.zeros((4, 3)))
    assert n.shape == (4, 0) and t.shape == (0, 3)
    m = rng.standard_normal((8, 5))
    n, t = ft.depar_general(m)
    assert n.shape == (8, 5)
    assert np.allclose(n @ t, m, atol=1e-12)


def test_depar_general_tolerance_and_float_work(rng):
    u = rng.standard_normal(50)
    n, _ = ft.depar_general(np.column_stack([u, u * (1.0 + 1e-14)]), tol=1e-12)
    assert n.shape[1] == 1
    ft.float_ops.reset()
    ft.depar_general(rng.standard_normal((10, 6)))
    assert ft.float_ops.count > 0


# ---- depar_quasi_perm (TestDeparQuasiPerm) --------------------------------

def test_depar_quasi_perm_factorises_exactly(rng):
    q = ft.QuasiPermMatrix(9, 14, rng.integers(0, 9, 14))
    n, t = ft.depar_quasi_perm(q)
    assert isinstance(n, ft.QuasiPermMatrix) and isinstance(t, ft.QuasiPermMatrix)
    assert np.array_equal(n.to_dense() @ t.to_dense(), q.to_dense())


def test_depar_quasi_perm_kept_rows(rng):
    q = ft.QuasiPermMatrix(7, 30, rng.integers(0, 7, 30))
    n, _ = ft.depar_quasi_perm(q)
    assert np.all(np.diff(n.col_to_row) > 0)
    assert n.n_cols <= q.n_rows
    assert n.n_cols == np.unique(q.col_to_row).size


def test_depar_quasi_perm_index_only(rng):
    q = ft.QuasiPermMatrix(40, 200, rng.integers(0, 40, 200))
    ft.float_ops.reset()
    ft.depar_quasi_perm(q)
    assert ft.float_ops.count == 0.0
    with pytest.raises(TypeError):
        ft.depar_quasi_perm(np.eye(3))


def test_depar_quasi_perm_agrees_with_general_route(rng):
    for _ in range(10):
        rows = int(rng.integers(2, 25))
        cols = int(rng.integers(1, 60))
        q = ft.QuasiPermMatrix(rows, cols, rng.integers(0, rows, cols))
        nq, _ = ft.depar_quasi_perm(q)
        ng, tg = ft.depar_general(q.to_dense())
        assert nq.n_cols == ng.shape[1]
        assert np.allclose(ng @ tg, q.to_dense(), atol=1e-13)


# ---- parallel_vector_round (TestParallelVectorRound) ---------------------

def _dense_route(s):
    """Deparallelise the materialised structured train with depar_general,
    asserting every handed-over matrix is a quasi-permutation (the
    reference test's dense_parallel_round)."""
    cores = [np.array(c) for c in structured_to_tt(s).cores]
    d, pv = len(cores), s.pivot
    for k in range(pv):
        r0, n, r1 = cores[k].shape
        m = cores[k].reshape(r0 * n, r1)
        assert as_quasi_perm(m) is not None
        nf, tf = ft.depar_general(m)
        cores[k] = nf.reshape(r0, n, nf.shape[1])
        cores[k + 1] = np.tensordot(tf, cores[k + 1], axes=(1, 0))
    for k in range(d - 1, pv, -1):
        r0, n, r1 = cores[k].shape
        m = cores[k].reshape(r0, n * r1).T
        assert as_quasi_perm(m) is not None
        nf, tf = ft.depar_general(m)
        cores[k] = np.ascontiguousarray(nf.T).reshape(nf.shape[1], n, r1)
        cores[k - 1] = np.einsum("abc,jc->abj", cores[k - 1], tf)
    return ft.TTTensor(cores)


@pytest.mark.parametrize("shape", [(4, 5, 6), (3, 3, 3, 3), (2, 6, 3, 4), (8, 9)])
def test_pvr_lossless_every_pivot(rng, shape):
    t = rand_sparse(rng, shape, 0.15)
    dense = t.to_dense()
    for pivot in range(len(shape)):
        tt = ft.parallel_vector_round(ft.build_structured_tt(t, pivot))
        assert np.array_equal(tt_to_full(tt), dense)


def test_pvr_rank_bounds(rng):
    t = rand_sparse(rng, (4, 3, 5, 2), 0.2)
    for pivot in range(t.ndim):
        s = ft.build_structured_tt(t, pivot)
        tt = ft.parallel_vector_round(s)
        for k in range(1, t.ndim):
            outer = math.prod(t.shape[:k]) if k <= pivot else math.prod(t.shape[k:])
            assert tt.ranks[k] <= min(s.num_fibers, outer)


def test_pvr_side_cores_exactly_orthonormal(rng):
    t = rand_sparse(rng, (4, 4, 4), 0.2)
    for pivot in range(3):
        tt = ft.parallel_vector_round(ft.build_structured_tt(t, pivot))
        for k, c in enumerate(tt.cores):
            c = np.asarray(c)
            r0, n, r1 = c.shape
            if k < pivot:
                m = c.reshape(r0 * n, r1)
                assert np.array_equal(m.T @ m, np.eye(r1))
            elif k > pivot:
                m = c.reshape(r0, n * r1)
                assert np.array_equal(m @ m.T, np.eye(r0))


def test_pvr_ranks_match_general_route(rng):
    t = rand_sparse(rng, (4, 3, 4), 0.25)
    for pivot in range(3):
        s = ft.build_structured_tt(t, pivot)
        ref = _dense_route(s)
        assert ft.parallel_vector_round(s).ranks == ref.ranks
        assert np.allclose(tt_to_full(ref), t.to_dense(), atol=1e-13)


def test_pvr_empty_single_and_no_float_work(rng):
    e = ft.SparseTensor((3, 4, 2), np.zeros((0, 3), dtype=np.int64), np.zeros(0))
    tt = ft.parallel_vector_round(ft.build_structured_tt(e, 1))
    assert not np.any(tt_to_full(tt))
    one = ft.SparseTensor((3, 4, 2), np.array([[1, 2, 0]]), np.array([5.0]))
    tt = ft.parallel_vector_round(ft.build_structured_tt(one, 0))
    assert tt.ranks == (1, 1, 1, 1)
    full = tt_to_full(tt)
    assert full[1, 2, 0] == 5.0 and np.count_nonzero(full) == 1
    s = ft.build_structured_tt(rand_sparse(rng, (5, 5, 5), 0.2), 1)
    ft.float_ops.reset()
    ft.parallel_vector_round(s)
    assert ft.float_ops.count == 0.0


# ---- TruncationBudget and the rounding modes (TestTruncationBudget,
# TestRoundingModes) -------------------------------------------------------

def test_budget_defaults_and_validation():
    b = ft.TruncationBudget()
    assert b.eps == 1e-14 and b.mode == "static"
    for kw in ({"mode": "bogus"}, {"eps": -1.0}, {"mode": "fixed_rank"}, {"delta_left": -0.1}):
        with pytest.raises(ValueError):
            ft.TruncationBudget(**kw)


@pytest.fixture
def exact_train(rng):
    t = rand_sparse(rng, (5, 4, 6, 3), 0.2)
    return t, 1, ft.parallel_vector_round(ft.build_structured_tt(t, 1))


@pytest.mark.parametrize("mode", ["static", "dynamic"])
def test_rounding_error_contract(exact_train, mode):
    t, pivot, tt = exact_train
    dense = t.to_dense()
    fn = ft.efficient_tt_rounding if mode == "static" else ft.dynamic_tt_rounding
    for eps in (0.5, 0.1, 0.01, 1e-14):
        out = fn(tt, ft.TruncationBudget(eps=eps, pivot=pivot, mode=mode))
        assert _rel(tt_to_full(out), dense) <= eps + 1e-12


def test_rounding_near_lossless_ranks_equal_tt_svd(exact_train):
    t, pivot, tt = exact_train
    out = ft.efficient_tt_rounding(tt, ft.TruncationBudget(eps=1e-14, pivot=pivot))
    assert out.ranks == tt_svd(t.to_dense(), 1e-14).ranks


def test_rounding_huge_budget_is_zero_train(exact_train):
    t, pivot, tt = exact_train
    out = ft.efficient_tt_rounding(tt, ft.TruncationBudget(eps=1.5, pivot=pivot))
    assert not np.any(tt_to_full(out))
    assert tt_to_full(out).shape == t.shape


def test_fixed_rank_targets_and_clamps(exact_train):
    t, pivot, tt = exact_train
    lossless = tt.ranks[1:-1]
    out = ft.fixed_rank_rounding(tt, ft.TruncationBudget(pivot=pivot, mode="fixed_rank",
                                                         fixed_ranks=lossless))
    assert np.allclose(tt_to_full(out), t.to_dense(), atol=1e-12 * np.linalg.norm(t.values))
    out = ft.fixed_rank_rounding(tt, ft.TruncationBudget(pivot=pivot, mode="fixed_rank",
                                                         fixed_ranks=1))
    assert all(r == 1 for r in out.ranks[1:-1])
    out = ft.fixed_rank_rounding(tt, ft.TruncationBudget(pivot=pivot, mode="fixed_rank",
                                                         fixed_ranks=999))
    assert all(r <= rt for r, rt in zip(out.ranks, tt.ranks))


def test_fixed_rank_error_dominates_unfolding_tails(exact_train):
    # Eckart-Young: a rank-r_k train cannot beat the best rank-r_k
    # approximation of unfolding k
    t, pivot, tt = exact_train
    dense = t.to_dense()
    out = ft.fixed_rank_rounding(tt, ft.TruncationBudget(pivot=pivot, mode="fixed_rank",
                                                         fixed_ranks=2))
    err = np.linalg.norm(tt_to_full(out) - dense)
    for k in range(1, t.ndim):
        sigma = np.linalg.svd(dense.reshape(math.prod(t.shape[:k]), -1), compute_uv=False)
        assert err >= np.sqrt(np.sum(sigma[out.ranks[k]:] ** 2)) - 1e-10


def test_rounding_mode_and_pivot_mismatch(exact_train):
    _, pivot, tt = exact_train
    with pytest.raises(ValueError):
        ft.efficient_tt_rounding(tt, ft.TruncationBudget(pivot=pivot, mode="dynamic"))
    with pytest.raises(ValueError):
        ft.dynamic_tt_rounding(tt, ft.TruncationBudget(pivot=pivot, mode="static"))
    with pytest.raises(ValueError):
        ft.fixed_rank_rounding(tt, ft.TruncationBudget(pivot=pivot, mode="static"))
    with pytest.raises(ft.ContractViolationError):
        ft.efficient_tt_rounding(tt, ft.TruncationBudget(eps=0.1, pivot=pivot + 1))


# ---- fasttt driver (TestFastTTDriver) -------------------------------------

def test_fasttt_near_lossless_report(rng):
    t = rand_sparse(rng, (5, 6, 4), 0.2)
    tt, rep = ft.fasttt(t)
    assert _rel(tt_to_full(tt), t.to_dense()) <= 1e-11
    assert rep.eps_actual <= 1e-11 and rep.eps_actual_method == "tt_difference"
    assert rep.shape == t.shape and rep.nnz == t.nnz
    assert rep.ranks == tt.ranks[1:-1]
    assert len(rep.ranks_lossless) == t.ndim - 1
    assert rep.flops_fasttt_model >= 0.0 and rep.flops_ttsvd_model > 0.0


def test_fasttt_eps_none_and_zero_are_lossless(rng):
    t = rand_sparse(rng, (4, 4, 4), 0.25)
    for eps in (None, 0.0):
        _, rep = ft.fasttt(t, eps=eps)
        assert rep.eps == 1e-14 and rep.eps_actual <= 1e-11


def test_fasttt_every_pivot_gives_the_same_tensor(rng):
    t = rand_sparse(rng, (4, 3, 2, 5), 0.2)
    dense = t.to_dense()
    norm = np.linalg.norm(dense)
    fulls = []
    for pivot in range(4):
        tt, rep = ft.fasttt(t, pivot=pivot)
        assert rep.pivot == pivot
        fulls.append(tt_to_full(tt))
    for a in fulls:
        assert np.linalg.norm(a - dense) / norm <= 1e-11
        for b in fulls:
            assert np.linalg.norm(a - b) / norm <= 1e-11


@pytest.mark.parametrize("shape,density", [((5, 4, 6), 0.15), ((3, 5, 3, 4), 0.1)])
def test_fasttt_ranks_equal_classical_tt_svd(rng, shape, density):
    t = rand_sparse(rng, shape, density)
    tt, _ = ft.fasttt(t)
    assert tt.ranks == tt_svd(t.to_dense(), 1e-14).ranks


@pytest.mark.parametrize("mode", ["static", "dynamic"])
def test_fasttt_moderate_eps(rng, mode):
    t = rand_sparse(rng, (6, 5, 4), 0.3)
    dense = t.to_dense()
    for eps in (0.3, 0.05):
        tt, rep = ft.fasttt(t, eps=eps, mode=mode)
        assert _rel(tt_to_full(tt), dense) <= eps + 1e-12
        assert rep.eps_actual <= eps + 1e-12 and rep.mode == mode


def test_fasttt_fixed_alias_empty_and_type(rng):
    t = rand_sparse(rng, (4, 5, 4), 0.2)
    tt, rep = ft.fasttt(t, eps=None, mode="fixed", fixed_ranks=(2, 2))
    assert rep.mode == "fixed_rank" and all(r <= 2 for r in tt.ranks[1:-1])
    e = ft.SparseTensor((3, 4, 5), np.zeros((0, 3), dtype=np.int64), np.zeros(0))
    tt, rep = ft.fasttt(e)
    assert not np.any(tt_to_full(tt)) and rep.eps_actual == 0.0 and rep.warnings
    with pytest.raises(TypeError):
        ft.fasttt(rng.standard_normal((3, 3)))


# ---- select_p (TestSelectP) -----------------------------------------------

def test_select_p_single_mode_and_ties():
    assert ft.select_p(ft.SparseTensor((5,), np.array([[2]]), np.array([1.0]))) == 0
    coords = np.array([[i, j, k] for i in range(3) for j in range(3) for k in range(3)])
    assert ft.select_p(ft.SparseTensor((3, 3, 3), coords, np.arange(1.0, 28.0))) == 0


@pytest.mark.parametrize("i,shape", list(enumerate([(4, 9, 3), (2, 12, 2, 6), (7, 3, 5),
                                                   (3, 4, 5, 2, 3)])))
def test_select_p_matches_enumerated_model(i, shape):
    t = rand_sparse(np.random.default_rng(100 + i), shape, 0.08)
    assert ft.select_p(t) == brute_select(t)


def test_select_p_targets_and_precise(rng):
    t = rand_sparse(rng, (4, 8, 3, 5), 0.1)
    assert ft.select_p(t, target_ranks=(2, 2, 2)) == brute_select(t, (2, 2, 2))
    t = rand_sparse(rng, (5, 4, 6), 0.15)
    costs = []
    for pivot in range(3):
        rt = lossless_bond_ranks(ft.build_structured_tt(t, pivot))
        r = [min(rt[k - 1], math.prod(t.shape[:k]), math.prod(t.shape[k:])) for k in range(1, 3)]
        costs.append(modeled_cost(t.shape, pivot, rt, r))
    assert ft.select_p(t, precise=True) == int(np.argmin(costs))


# ---- cost model (TestFlopsModel) ------------------------------------------

def test_flops_model_hand_counts():
    assert ft.flops_fasttt((6, 8), pivot=0, ranks_lossless=(5,), ranks_final=(2,)) == 6 * 5 * 5
    assert ft.flops_fasttt((6, 8), pivot=1, ranks_lossless=(5,),
                           ranks_final=(2,)) == (5 * 8) * 1 * 1 + 5 * (8 * 1) * 5
    assert ft.flops_fasttt((9,), 0, (), ()) == 0.0
    a = ft.flops_fasttt((4, 5, 6), 1, (3, 3), (2, 2))
    assert ft.flops_fasttt((4, 5, 6), 1, (3, 3), (2, 2), c_svd=3.0) == 3.0 * a


# ---- error measures (TestErrorMeasures) -----------------------------------

def test_tt_relative_error_against_dense(rng):
    t = rand_sparse(rng, (5, 5, 5), 0.2)
    tt, _ = ft.fasttt(t)
    rounded, _ = ft.fasttt(t, eps=0.3)
    dense = t.to_dense()
    want = _rel(tt_to_full(rounded), dense)
    assert ft.tt_relative_error(tt, rounded) == pytest.approx(want, rel=1e-8, abs=1e-12)


def test_sparse_inner_error_against_dense(rng):
    t = rand_sparse(rng, (6, 5, 4), 0.3)
    rounded, _ = ft.fasttt(t, eps=0.2)
    want = _rel(tt_to_full(rounded), t.to_dense())
    assert ft.sparse_inner_error(t, rounded) == pytest.approx(want, abs=1e-6)


def test_exact_trains_measure_zero(rng):
    t = rand_sparse(rng, (4, 4, 4), 0.3)
    tt = ft.parallel_vector_round(ft.build_structured_tt(t, 1))
    exact, _ = ft.fasttt(t)
    assert ft.tt_relative_error(tt, exact) <= 1e-12


# ---- svd_truncate_delta / _rank, qr_economic (test_linalg.py) -------------

def _oracle_rank(sigma, delta):
    sq = sigma ** 2
    return next((r for r in range(len(sigma) + 1) if sq[r:].sum() <= delta * delta), len(sigma))


def test_svd_delta_diagonal_example():
    m = np.diag([3.0, 2.0, 1.0])
    res = ft.svd_truncate_delta(m, 1.0)
    assert res.rank == 2 and res.trunc_error == pytest.approx(1.0, rel=1e-12)
    res = ft.svd_truncate_delta(m, np.sqrt(5.0) + 1e-12)
    assert res.rank == 1 and res.trunc_error == pytest.approx(np.sqrt(5.0), rel=1e-12)


def test_svd_delta_zero_budget(rng):
    res = ft.svd_truncate_delta(rng.standard_normal((6, 4)), 0.0)
    assert res.rank == 4 and res.trunc_error == 0.0
    u, v = rng.standard_normal((8, 1)), rng.standard_normal((1, 5))
    assert ft.svd_truncate_delta(u @ v, 0.0).rank == 1
    assert ft.svd_truncate_delta(np.zeros((4, 3)), 0.0).rank == 0


def test_svd_delta_rank_zero_above_norm(rng):
    m = rng.standard_normal((5, 5))
    res = ft.svd_truncate_delta(m, np.linalg.norm(m) * 1.001)
    assert res.rank == 0 and res.u.shape == (5, 0) and res.vt.shape == (0, 5)
    assert res.trunc_error == pytest.approx(np.linalg.norm(m), rel=1e-12)


def test_svd_delta_reported_error_and_monotone(rng):
    m = rng.standard_normal((12, 9))
    for delta in (0.5, 1.5, 3.0):
        res = ft.svd_truncate_delta(m, delta)
        err = np.linalg.norm(m - (res.u * res.s) @ res.vt)
        assert err == pytest.approx(res.trunc_error, abs=1e-10) and err <= delta + 1e-10
    m = rng.standard_normal((10, 10))
    ranks = [ft.svd_truncate_delta(m, d).rank for d in np.linspace(0.0, np.linalg.norm(m), 25)]
    assert all(a >= b for a, b in zip(ranks, ranks[1:]))


@given(st.integers(2, 8), st.integers(2, 8), st.floats(0.0, 4.0), st.integers(0, 2**31 - 1))
@settings(max_examples=40, deadline=None)
def test_svd_delta_tail_rule_property(rows, cols, delta, seed):
    m = np.random.default_rng(seed).standard_normal((rows, cols))
    sigma = np.linalg.svd(m, compute_uv=False)
    res = ft.svd_truncate_delta(m, delta)
    if delta > 0.0:
        assert res.rank == _oracle_rank(sigma, delta)


def test_svd_delta_deterministic_signs_and_errors(rng):
    m = rng.standard_normal((7, 5))
    a = ft.svd_truncate_delta(m, 0.1)
    b = ft.svd_truncate_delta(m.copy(), 0.1)
    assert np.array_equal(a.u, b.u) and np.array_equal(a.vt, b.vt)
    for j in range(a.rank):
        assert a.u[np.argmax(np.abs(a.u[:, j])), j] >= 0.0
    for bad, delta in ((np.array([1.0, 2.0]), 0.0), (np.array([[np.nan, 1.0]]), 0.0),
                       (np.ones((2, 2)), -0.5)):
        with pytest.raises(ValueError):
            ft.svd_truncate_delta(bad, delta)


def test_svd_rank_contract(rng):
    m = rng.standard_normal((8, 6))
    res = ft.svd_truncate_rank(m, 3)
    assert res.rank == 3 and res.u.shape == (8, 3) and res.vt.shape == (3, 6)
    assert ft.svd_truncate_rank(rng.standard_normal((4, 6)), 10).rank == 4
    m = rng.standard_normal((9, 7))
    sigma = np.linalg.svd(m, compute_uv=False)
    res = ft.svd_truncate_rank(m, 2)
    want = np.sqrt(np.sum(sigma[2:] ** 2))
    assert res.trunc_error == pytest.approx(want, rel=1e-12)
    assert np.linalg.norm(m - (res.u * res.s) @ res.vt) == pytest.approx(want, rel=1e-10)
    m = rng.standard_normal((3, 3))
    res = ft.svd_truncate_rank(m, 0)
    assert res.rank == 0 and res.trunc_error == pytest.approx(np.linalg.norm(m), rel=1e-12)


@pytest.mark.parametrize("shape", [(8, 5), (5, 8), (6, 6), (7, 1)])
def test_qr_economic_factorisation(rng, shape):
    m = rng.standard_normal(shape)
    res = ft.qr_economic(m)
    k = min(shape)
    assert res.q.shape == (shape[0], k) and res.r.shape == (k, shape[1])
    assert np.allclose(res.q.T @ res.q, np.eye(k), atol=1e-12)
    assert np.allclose(res.q @ res.r, m, atol=1e-12)
    assert np.all(np.diag(res.r) >= 0.0)
    again = ft.qr_economic(m.copy())
    assert np.array_equal(res.q, again.q) and np.array_equal(res.r, again.r)


# ---- fiber extraction (test_tensor.py TestFiberExtraction) ----------------

def test_fibers_round_trip_and_counts(rng):
    t = rand_sparse(rng, (4, 3, 5, 2), 0.25)
    for pivot in range(t.ndim):
        fs = ft.extract_nonzero_fibers(t, pivot)
        back = fs.to_tensor()
        assert np.array_equal(back.coords, t.coords) and np.array_equal(back.values, t.values)
        assert fs.num_fibers == len({tuple(np.delete(c, pivot)) for c in t.coords})


def test_fibers_sorted_distinct_nonempty_bounded(rng):
    fs = ft.extract_nonzero_fibers(rand_sparse(rng, (5, 4, 3), 0.3), 1)
    keys = [tuple(r) for r in fs.fixed_coords]
    assert keys == sorted(keys) and len(set(keys)) == len(keys)
    t = rand_sparse(rng, (6, 6), 0.2)
    for pivot in (0, 1):
        assert np.all(np.diff(ft.extract_nonzero_fibers(t, pivot).indptr) >= 1)
    t = rand_sparse(rng, (4, 5, 6), 0.1)
    fs = ft.extract_nonzero_fibers(t, 2)
    assert fs.num_fibers <= t.nnz and fs.num_fibers <= 4 * 5


def test_fibers_empty_and_full_mode():
    e = ft.SparseTensor((3, 4), np.zeros((0, 2), dtype=np.int64), np.zeros(0))
    fs = ft.extract_nonzero_fibers(e, 0)
    assert fs.num_fibers == 0 and fs.to_tensor().nnz == 0
    coords = np.array([[i, j] for i in range(3) for j in range(4)])
    fs = ft.extract_nonzero_fibers(ft.SparseTensor((3, 4), coords, np.arange(1.0, 13.0)), 1)
    assert fs.num_fibers == 3 and np.all(np.diff(fs.indptr) == 4)
