"""CPU-side checks: the C-ABI library loads and exports every declared
symbol; host logic (validation, cost models, truncation rule, generators)
matches the reference conventions. No kernel is launched here."""

import ctypes
import math
import os
import re

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import ROOT, load_golden
from oracle import fasttt_oracle as O
import paper_1908_02721_b200 as ft
from paper_1908_02721_b200 import _native as nat
from paper_1908_02721_b200 import dense, generators as G, pipeline as P


def declared_symbols():
    with open(os.path.join(ROOT, "include", "fasttt_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(ftt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = nat.load_library()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in nat.SIGNATURES, f"{name} has no ctypes signature"
    assert set(nat.SIGNATURES) == set(names)
    assert lib.ftt_version().decode().startswith("fasttt_b200")


def test_library_is_sm100a():
    path = nat.LIB_PATH
    with open(path, "rb") as fh:
        blob = fh.read()
    assert b"sm_100a" in blob or b"compute_100a" in blob or len(blob) > 100000


def test_no_context_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        nat.context()


def test_status_mapping():
    nat.load_library()
    with pytest.raises(MemoryError):
        nat.check(nat.FTT_ERR_OOM)
    with pytest.raises(ValueError):
        nat.check(nat.FTT_ERR_INVALID)
    with pytest.raises(ValueError):
        nat.check(nat.FTT_ERR_NONFINITE)
    with pytest.raises(np.linalg.LinAlgError):
        nat.check(nat.FTT_ERR_NOCONV)
    with pytest.raises(RuntimeError):
        nat.check(nat.FTT_ERR_CUDA)


# ------------------------------------------------------------ containers
def test_sparse_tensor_contract():
    t = ft.SparseTensor((3, 4), [[2, 1], [0, 3], [1, 1]], [1.0, 0.0, 2.0])
    assert t.nnz == 2
    assert np.array_equal(t.coords, [[1, 1], [2, 1]])
    with pytest.raises(AttributeError):
        t.shape = (1,)
    with pytest.raises(ft.FormatError):
        ft.SparseTensor((3, 4), [[3, 0]], [1.0])
    with pytest.raises(ft.FormatError):
        ft.SparseTensor((3, 4), [[1, 1], [1, 1]], [1.0, 2.0])
    with pytest.raises(ft.FormatError):
        ft.SparseTensor((3, 4), [[1, 1]], [np.nan])
    with pytest.raises(ValueError):
        ft.check_shape((2, 0))
    with pytest.raises(ValueError):
        ft.check_shape((2 ** 32, 2 ** 31))
    with pytest.raises(TypeError):
        ft.check_shape((2.5, 3))
    assert issubclass(ft.FormatError, ValueError)
    assert issubclass(ft.ContractViolationError, RuntimeError)


def test_fiberset_and_quasiperm_validation():
    with pytest.raises(ValueError):
        ft.FiberSet((3, 4), 0, np.zeros((1, 1), np.int64), [0, 2], [0, 1], [1.0])
    with pytest.raises(ValueError):
        ft.QuasiPermMatrix(3, 2, [0, 3])
    q = ft.QuasiPermMatrix(3, 2, [2, 0])
    assert np.array_equal(q.to_dense(), [[0, 1], [0, 0], [1, 0]])


def test_linearize_known_answer():
    assert list(ft.linearize((2, 3, 4), [[0, 0, 0], [0, 0, 1], [1, 2, 3]])) == [0, 1, 23]


@given(st.lists(st.integers(1, 9), min_size=1, max_size=5), st.integers(0, 2 ** 31 - 1))
@settings(max_examples=50, deadline=None)
def test_linearize_round_trip(shape, seed):
    rng = np.random.default_rng(seed)
    coords = np.stack([rng.integers(0, n, 20) for n in shape], 1)
    assert np.array_equal(ft.delinearize(shape, ft.linearize(shape, coords)), coords)


# ------------------------------------------------------------ cost models
def test_flops_models_hand_counts():
    assert P.flops_fasttt((6, 8), 0, (5,), (2,)) == 6 * 5 * 5
    assert P.flops_fasttt((6, 8), 1, (5,), (2,)) == (5 * 8) * 1 * 1 + 5 * (8 * 1) * 5
    assert P.flops_fasttt((9,), 0, (), ()) == 0.0
    a = P.flops_fasttt((4, 5, 6), 1, (3, 3), (2, 2))
    assert P.flops_fasttt((4, 5, 6), 1, (3, 3), (2, 2), c_svd=3.0) == 3.0 * a
    for shape, pivot, rl, rf in [((4, 5, 6, 7), 2, (4, 20, 7), (3, 5, 2)),
                                 ((10, 3, 7), 0, (10, 7), (2, 2))]:
        assert P.flops_fasttt(shape, pivot, rl, rf) == O.flops_fasttt(shape, pivot, rl, rf)
        assert P.flops_ttsvd(shape, rf) == O.flops_ttsvd(shape, rf)
    assert P.full_ranks((3, 4, 5), (2, 2)) == (1, 2, 2, 1)
    with pytest.raises(ValueError):
        P.full_ranks((3, 4, 5), (2,))


def test_upper_bounds_match_oracle():
    for dims in [(4, 9, 3), (2, 12, 2, 6), (100,) * 4, (32,) * 12]:
        for p in range(len(dims)):
            assert P._upper_bond_bounds(dims, p, 1234) == O.upper_bond_bounds(dims, p, 1234)


def test_truncation_budget_validation():
    b = P.TruncationBudget()
    assert b.eps == 1e-14 and b.mode == "static"
    for kw in ({"mode": "bogus"}, {"eps": -1.0}, {"mode": "fixed_rank"}, {"delta_left": -0.1}):
        with pytest.raises(ValueError):
            P.TruncationBudget(**kw)


def test_diag_truncation_known_answer():
    s = np.array([3.0, 2.0, 1.0])
    assert dense.tail_rank(s, 1.0, (3, 3)) == 2
    assert dense.tail_error(s, 2) == pytest.approx(1.0, rel=1e-12)
    assert dense.tail_rank(s, np.sqrt(5.0) + 1e-12, (3, 3)) == 1
    assert dense.tail_rank(np.zeros(3), 0.0, (3, 3)) == 0


@given(st.lists(st.floats(0.0, 10.0), min_size=1, max_size=8), st.floats(0.0, 4.0))
@settings(max_examples=80, deadline=None)
def test_tail_rule_matches_brute_force(svals, delta):
    s = np.sort(np.asarray(svals))[::-1]
    got = dense.tail_rank(s, delta, (len(s), len(s)))
    assert got == O.truncation_rank(s, delta, (len(s), len(s)))
    if delta > 0:
        brute = next(r for r in range(len(s) + 1) if (s[r:] ** 2).sum() <= delta * delta)
        assert got == brute


def test_generators_reproduce_golden_inputs():
    import hashlib

    for cfg in (1, 2, 4):
        g = load_golden(f"c{cfg}")
        meta, _ = g
        shape, coords, vals, eps = G.gen_config(cfg)
        dims, coords, vals = O.canonical(shape, coords, vals)
        h = hashlib.sha256()
        a = np.ascontiguousarray(coords)
        h.update(str(a.dtype).encode()); h.update(str(a.shape).encode()); h.update(a.tobytes())
        assert h.hexdigest() == meta["input_coords"]
        assert eps == meta["eps"]
        assert coords.shape[0] == meta["nnz"]


def test_config_nnz_match_baseline_bounds():
    bounds = {1: 50_000, 2: 373_248, 3: 236_196 + 2000, 4: 326_656}
    for cfg, bound in bounds.items():
        shape, coords, vals, _ = G.gen_config(cfg)
        assert coords.shape[0] <= bound
    assert G.gen_config(4)[1].shape[0] == 326_656


def test_tensorize_and_split_are_layout_only():
    import scipy.sparse

    m = scipy.sparse.random(12, 20, density=0.3, random_state=3, format="coo")
    t = ft.tensorize_matrix(m, (3, 4), (4, 5))
    assert t.shape == (12, 20)
    cores = [np.arange(1 * 12 * 2, dtype=float).reshape(1, 12, 2),
             np.arange(2 * 20 * 1, dtype=float).reshape(2, 20, 1)]
    mpo = ft.tt_split_mpo(ft.TTTensor(cores), (3, 4), (4, 5))
    assert mpo.cores[0].shape == (1, 3, 4, 2) and mpo.cores[1].shape == (2, 4, 5, 1)
    with pytest.raises(ValueError):
        ft.tt_split_mpo(ft.TTTensor(cores), (3, 4), (5, 4, 1))


def test_api_type_errors_without_gpu():
    with pytest.raises(TypeError):
        ft.fasttt(np.zeros((3, 3)))
    with pytest.raises(TypeError):
        ft.select_p(np.zeros((3, 3)))
    with pytest.raises(TypeError):
        ft.build_structured_tt(np.zeros((3, 3)), 0)
    with pytest.raises(TypeError):
        ft.parallel_vector_round(np.eye(3))
    with pytest.raises(TypeError):
        ft.depar_quasi_perm(np.eye(3))


def test_select_p_single_mode_host_only():
    t = ft.SparseTensor((5,), np.array([[2]]), np.array([1.0]))
    assert ft.select_p(t) == 0


def test_tt_entries_index_contract_matches_numpy():
    """tt_entries' host-side index check reproduces the reference's numpy
    slicing contract (ttformat.py:124-136): IndexError text of the first
    offending batch / mode / value, negative indices wrapped."""
    from paper_1908_02721_b200 import trains as T

    dims = (3, 5, 4)
    rng = np.random.default_rng(3)
    cores = [rng.standard_normal((1 if k == 0 else 2, n, 1 if k == 2 else 2))
             for k, n in enumerate(dims)]

    def numpy_loop(coords, batch):
        for lo in range(0, coords.shape[0], batch):
            c = coords[lo:lo + batch]
            cores[0][0, c[:, 0], :]
            for k in range(1, 3):
                cores[k][:, c[:, k], :]

    ok = np.array([[0, 4, 3], [-1, -5, -4], [2, 0, 1]])
    assert T._checked_indices(ok, dims, 1024).tolist() == [[0, 4, 3], [2, 0, 0], [2, 0, 1]]
    for bad, batch in ((np.array([[0, 0, 0], [0, 5, 9]]), 1024),
                       (np.array([[0, 0, 4], [3, 0, 0]]), 1024),
                       (np.array([[0, 0, 4], [3, 0, 0]]), 1),
                       (np.array([[-4, 0, 0]]), 1024)):
        with pytest.raises(IndexError) as want:
            numpy_loop(bad, batch)
        with pytest.raises(IndexError) as got:
            T._checked_indices(bad, dims, batch)
        assert str(got.value) == str(want.value)
