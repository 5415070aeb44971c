"""Pins the CPU oracle (oracle/fasttt_oracle.py) to the reference.

The golden fixtures were produced by the unmodified reference
(tests/golden/make_golden.py). Integer outputs must match bit-exactly;
reconstructions within 1e-10 relative Frobenius error.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle import fasttt_oracle as O
from paper_1908_02721_b200 import generators as G


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def _small():
    with open(os.path.join(GOLDEN, "small.json")) as fh:
        cases = json.load(fh)
    return cases, np.load(os.path.join(GOLDEN, "small.npz"))


def test_small_suite_matches_reference():
    cases, z = _small()
    nruns = 0
    for case in cases:
        if case["id"] == "d1":
            assert case["fasttt"].startswith("ValueError")
            continue
        i = case["id"]
        shape = tuple(case["shape"])
        coords, values = z[f"t{i}_coords"], z[f"t{i}_values"]
        assert O.select_p(shape, coords, values) == case["select_p"]
        assert O.select_p(shape, coords, values, precise=True) == case["select_p_precise"]
        assert O.select_p(shape, coords, values, target_ranks=2) == case["select_p_target2"]
        for p in range(len(shape)):
            fb = O.extract_fibers(shape, coords, values, p)
            assert np.array_equal(fb["fixed_coords"], z[f"t{i}_p{p}_fixed"])
            assert np.array_equal(fb["indptr"], z[f"t{i}_p{p}_indptr"])
            assert np.array_equal(fb["pivot_index"], z[f"t{i}_p{p}_pidx"])
            assert np.array_equal(fb["values"], z[f"t{i}_p{p}_fvals"])
        for run in case["runs"]:
            cores, info = O.fasttt(shape, coords, values, eps=run["eps"], pivot=run["pivot"],
                                   mode=run["mode"], **run["kw"])
            assert list(info["ranks"]) == run["ranks"], run["tag"]
            assert list(info["ranks_lossless"]) == run["ranks_lossless"]
            assert info["num_fibers"] == run["num_fibers"]
            ref = [z[f"{run['tag']}_core{k}"] for k in range(len(shape))]
            probe = np.concatenate([coords, G.zero_positions(shape, coords, 64, seed=5)])
            a, b = O.tt_entries(cores, probe), O.tt_entries(ref, probe)
            nb = np.linalg.norm(b)
            assert np.linalg.norm(a - b) <= 1e-10 * max(nb, 1e-300) or nb == 0.0
            assert info["eps_actual_method"] == run["eps_actual_method"]
            assert abs(info["eps_actual"] - run["eps_actual"]) <= 1e-9
            nruns += 1
    assert nruns >= 200


def test_d1_raises_like_reference():
    cases, z = _small()
    case = [c for c in cases if c["id"] == "d1"][0]
    assert "inconsistent fiber index pointers" in case["fasttt"]


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_config_goldens(cfg):
    g = load_golden(f"c{cfg}")
    assert g is not None
    meta, z = g
    shape, coords, vals, eps = G.gen_config(cfg)
    dims, coords, vals = O.canonical(shape, coords, vals)
    assert digest(coords) == meta["input_coords"]
    assert digest(vals) == meta["input_values"]
    counts = [O.fiber_count(dims, coords, p) for p in range(len(dims))]
    assert counts == meta["fiber_counts"]
    p = O.select_p(dims, coords, vals)
    assert p == meta["auto_pivot"]
    idx = meta["index"]
    fb = O.extract_fibers(dims, coords, vals, p)
    assert digest(fb["fixed_coords"]) == idx["fixed_coords"]
    assert digest(fb["indptr"]) == idx["indptr"]
    assert digest(fb["pivot_index"]) == idx["pivot_index"]
    assert digest(fb["values"]) == idx["fiber_values"]
    left, t_map, r_prev, right, s_map, r_next = O.index_sweeps(dims, p, fb["fixed_coords"])
    assert [digest(k) for k, _ in left] == idx["left_kept"]
    assert [digest(k) for k, _ in right] == idx["right_kept"]
    assert digest(t_map) == idx["t_map"] and digest(s_map) == idx["s_map"]
    cores, info = O.fasttt(dims, coords, vals, eps=eps, report=False)
    assert list(info["ranks"]) == meta["ranks"]
    a = np.concatenate([O.tt_entries(cores, coords), O.tt_entries(cores, z["zero_coords"])])
    b = np.concatenate([z["entries_nnz"], z["entries_zero"]])
    assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
    if meta.get("mid_pivot") is not None:
        assert meta["mid_ranks_ref"] == meta["mid_ranks_oracle"]


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [3, 5])
def test_config_goldens_large_index(cfg):
    """c3/c5: integer goldens from the reference's own index functions."""
    g = load_golden(f"c{cfg}")
    if g is None:
        pytest.skip(f"c{cfg} golden not generated yet")
    meta, _ = g
    shape, coords, vals, eps = G.gen_config(cfg)
    dims, coords, vals = O.canonical(shape, coords, vals)
    assert digest(coords) == meta["input_coords"]
    p = meta["auto_pivot"]
    idx = meta["index"]
    fb = O.extract_fibers(dims, coords, vals, p)
    assert digest(fb["indptr"]) == idx["indptr"]
    assert digest(fb["fixed_coords"]) == idx["fixed_coords"]
    left, t_map, r_prev, right, s_map, r_next = O.index_sweeps(dims, p, fb["fixed_coords"])
    assert [digest(k) for k, _ in left] == idx["left_kept"]
    assert [digest(k) for k, _ in right] == idx["right_kept"]
    assert list(O.lossless_bond_ranks(dims, p, left, right)) == idx["ranks_lossless"]


# ---- known answers pinned by the reference's own unit tests
def test_known_answers():
    assert list(O.linearize((2, 3, 4), [[0, 0, 0], [0, 0, 1], [1, 2, 3]])) == [0, 1, 23]
    u, s, vt, rank, err = O.svd_truncate_delta(np.diag([3.0, 2.0, 1.0]), 1.0)
    assert rank == 2 and abs(err - 1.0) < 1e-12
    assert O.flops_fasttt((6, 8), 0, (5,), (2,)) == 6 * 5 * 5
    assert O.flops_fasttt((6, 8), 1, (5,), (2,)) == (5 * 8) * 1 * 1 + 5 * (8 * 1) * 5
    coords = np.array([[i, j, k] for i in range(3) for j in range(3) for k in range(3)])
    assert O.select_p((3, 3, 3), coords, np.arange(1.0, 28.0)) == 0
