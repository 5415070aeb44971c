"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference.

Run in the build container only (it imports ``sparsett`` from
``/root/reference/pkg/src``; that tree does not exist on the GPU box, which
only reads the committed ``.npz`` / ``.json`` files)::

    python tests/golden/make_golden.py small c1 c2 c4 c3 c5

What comes from where:

* ``small``: 24 seeded small tensors x every pivot x 3 modes, run through the
  reference ``fasttt`` -- cores, ranks, report fields, fiber arrays.
* c1: the reference ``fasttt(a, eps)`` at its own auto pivot.
* c3: index goldens from the reference, train from the oracle (the reference's
  own run at the auto pivot did not finish in > 3 h here; ``REF_C3=1`` runs it).
* c2, c4, c5: the reference raises MemoryError at the auto pivot (it
  densifies the 0/1 cores, fasttt.py:246-255). Their integer goldens (pivot,
  per-pivot fiber counts, FiberSet, kept arrays, maps, lossless ranks) come
  from the reference's own index-only functions (``select_p``,
  ``build_structured_tt``, ``_index_sweeps``); c2 and c4 are additionally run
  end to end by the reference at an explicit middle pivot (c2 p=2, c4 p=3)
  and the oracle is checked against that; the final train at the auto pivot
  comes from the oracle restatement (oracle/fasttt_oracle.py), which is
  bit-identical to the reference wherever both run.
"""

from __future__ import annotations

import hashlib
import importlib
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import sparsett  # noqa: E402  (the reference)
from oracle import fasttt_oracle as O  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402

REF_FT = importlib.import_module("sparsett.fasttt")
ZERO_SAMPLES = 20_000
CORE_STORE_CAP = 400_000  # store full cores when the train is this small


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def index_goldens(t, pivot):
    """Integer outputs from the reference's own index-only functions."""
    s = sparsett.build_structured_tt(t, pivot)
    f = s.fibers
    left, t_map, r_prev, right, s_map, r_next = REF_FT._index_sweeps(s)
    g = {
        "pivot": int(pivot),
        "num_fibers": int(s.num_fibers),
        "ranks_lossless": [int(x) for x in REF_FT._lossless_bond_ranks(s)],
        "fixed_coords": digest(f.fixed_coords),
        "indptr": digest(f.indptr),
        "pivot_index": digest(f.pivot_index),
        "fiber_values": digest(f.values),
        "t_map": digest(t_map),
        "s_map": digest(s_map),
        "left_kept": [digest(k) for k, _ in left],
        "right_kept": [digest(k) for k, _ in right],
        "r_prev": int(r_prev),
        "r_next": int(r_next),
    }
    return g


def fiber_counts(t):
    d = t.ndim
    out = []
    for p in range(d):
        rest = [k for k in range(d) if k != p]
        keys = sparsett.tensor.linearize(tuple(t.shape[k] for k in rest), t.coords[:, rest])
        out.append(int(np.unique(keys).size))
    return out


def save_config(name, t, eps, cores, meta, zero_seed=12345):
    zc = G.zero_positions(t.shape, t.coords, ZERO_SAMPLES, seed=zero_seed)
    arrays = {"zero_coords": zc}
    nparam = sum(c.size for c in cores)
    if nparam <= CORE_STORE_CAP:
        for k, c in enumerate(cores):
            arrays[f"core{k}"] = c
        meta["cores_stored"] = True
    else:
        meta["cores_stored"] = False
    arrays["entries_nnz"] = O.tt_entries(cores, t.coords)
    arrays["entries_zero"] = O.tt_entries(cores, zc)
    meta["input_coords"] = digest(t.coords)
    meta["input_values"] = digest(t.values)
    meta["nnz"] = int(t.nnz)
    meta["shape"] = list(t.shape)
    meta["eps"] = eps
    meta["ranks"] = [int(c.shape[2]) for c in cores[:-1]]
    meta["ref_norm"] = float(O.tt_norm(cores))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(name, json.dumps({k: meta[k] for k in ("ranks", "nnz")}), flush=True)


def config(cfg: int):
    shape, coords, vals, eps = G.gen_config(cfg, seed=0)
    t = sparsett.SparseTensor(shape, coords, vals)
    meta = {"config": cfg, "seed": 0, "generator": G.CONFIGS[cfg]["name"]}
    t0 = time.time()
    meta["fiber_counts"] = fiber_counts(t)
    p = sparsett.select_p(t)
    meta["select_p_s"] = time.time() - t0
    meta["auto_pivot"] = int(p)
    meta["index"] = index_goldens(t, p)
    # c3: the reference fasttt() at its auto pivot densifies two 0/1 cores and
    # ran > 3 h in the 16-core build container without finishing; its train is
    # taken from the oracle restatement (bit-identical to the reference where
    # both run, c1 and the small suite) -- set REF_C3=1 to run the reference.
    ref_full = cfg == 1 or (cfg == 3 and os.environ.get("REF_C3") == "1")
    if ref_full:
        t0 = time.time()
        tt, rep = sparsett.fasttt(t, eps=eps)
        meta["ref_fasttt_s"] = time.time() - t0
        meta["source"] = "reference fasttt() at auto pivot"
        meta["report"] = {"eps_actual": rep.eps_actual, "method": rep.eps_actual_method,
                          "eps_actual_inner": rep.eps_actual_inner,
                          "flops_fasttt_model": rep.flops_fasttt_model,
                          "flops_ttsvd_model": rep.flops_ttsvd_model}
        cores = [np.array(c) for c in tt.cores]
    else:
        if cfg in (2, 4):
            mid = {2: 2, 4: 3}[cfg]
            t0 = time.time()
            s = sparsett.build_structured_tt(t, mid)
            ex = sparsett.parallel_vector_round(s)
            rt = sparsett.efficient_tt_rounding(
                ex, sparsett.TruncationBudget(eps=eps, pivot=mid, mode="static"))
            meta["ref_mid_pivot_s"] = time.time() - t0
            oc, oi = O.fasttt(t.shape, t.coords, t.values, eps=eps, pivot=mid, report=False)
            meta["mid_pivot"] = mid
            meta["mid_ranks_ref"] = [int(c.shape[2]) for c in rt.cores[:-1]]
            meta["mid_ranks_oracle"] = list(oi["ranks"])
            meta["mid_max_core_diff"] = max(float(np.abs(a - b).max()) for a, b in zip(rt.cores, oc))
            del s, ex, rt
        t0 = time.time()
        cores, info = O.fasttt(t.shape, t.coords, t.values, eps=eps, pivot=p, report=False)
        meta["oracle_s"] = time.time() - t0
        meta["source"] = ("oracle restatement at auto pivot (reference OOM or > 3 h there); "
                          "index goldens from reference")
        assert list(info["ranks_lossless"]) == meta["index"]["ranks_lossless"]
    save_config(f"c{cfg}", t, eps, cores, meta)


def config5_index():
    """Config 5 (8.5M nonzeros, 32^12): the reference cannot decompose it at
    any pivot within this container's memory (the dense pivot core alone is
    10.5 GB at p = 2, fasttt.py:253), so its golden is the reference's own
    INDEX path -- per-pivot fiber counts, select_p, FiberSet / kept / map
    digests, lossless ranks -- plus seeded zero positions.  The float check
    on the GPU is size-independent: a sum of 16 generic rank-1 terms has
    every unfolding rank 16, so the train must have ranks (16,)*11 and
    reproduce the input at every nonzero and 0 at the zero positions
    (tests/test_gpu_parity.py::test_config5_parity)."""
    shape, coords, vals, eps = G.gen_config(5, seed=0)
    t = sparsett.SparseTensor(shape, coords, vals)
    meta = {"config": 5, "seed": 0, "generator": G.CONFIGS[5]["name"]}
    t0 = time.time()
    meta["fiber_counts"] = fiber_counts(t)
    p = sparsett.select_p(t)
    meta["select_p_s"] = time.time() - t0
    meta["auto_pivot"] = int(p)
    t0 = time.time()
    meta["index"] = index_goldens(t, p)
    meta["index_s"] = time.time() - t0
    meta["input_coords"] = digest(t.coords)
    meta["input_values"] = digest(t.values)
    meta["nnz"] = int(t.nnz)
    meta["shape"] = list(t.shape)
    meta["eps"] = eps
    meta["source"] = ("reference index-only functions (select_p, build_structured_tt, "
                      "_index_sweeps); float check by construction (rank-16 sum)")
    zc = G.zero_positions(t.shape, t.coords, ZERO_SAMPLES, seed=12345)
    np.savez_compressed(os.path.join(HERE, "c5idx.npz"), zero_coords=zc)
    with open(os.path.join(HERE, "c5idx.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("c5idx", meta["auto_pivot"], meta["index"]["ranks_lossless"], flush=True)


def rand_sparse(rng, shape, density):
    size = math.prod(shape)
    nnz = int(density * size)
    lin = np.sort(rng.permutation(size)[:nnz].astype(np.int64))
    vals = rng.uniform(-1.0, 1.0, nnz)
    vals[vals == 0.0] = 0.5
    return sparsett.SparseTensor(shape, sparsett.tensor.delinearize(shape, lin), vals)


SMALL_SHAPES = [(4, 5, 6), (3, 3, 3, 3), (2, 6, 3, 4), (8, 9), (5, 4, 6, 3), (7, 2),
                (6, 5, 4), (3, 5, 3, 4), (4, 3, 2, 5), (2, 2, 2, 2, 2), (10, 3, 7), (3, 12, 2)]


def small():
    rng = np.random.default_rng(20261020)
    arrays = {}
    cases = []
    for i, shape in enumerate(SMALL_SHAPES * 2):
        dens = 0.25 if i < len(SMALL_SHAPES) else 0.08
        t = rand_sparse(rng, shape, dens)
        arrays[f"t{i}_coords"] = t.coords
        arrays[f"t{i}_values"] = t.values
        case = {"id": i, "shape": list(shape), "select_p": int(sparsett.select_p(t)),
                "select_p_precise": int(sparsett.select_p(t, precise=True)),
                "select_p_target2": int(sparsett.select_p(t, target_ranks=2)),
                "runs": []}
        for p in range(len(shape)):
            fs = sparsett.extract_nonzero_fibers(t, p)
            arrays[f"t{i}_p{p}_fixed"] = fs.fixed_coords
            arrays[f"t{i}_p{p}_indptr"] = fs.indptr
            arrays[f"t{i}_p{p}_pidx"] = fs.pivot_index
            arrays[f"t{i}_p{p}_fvals"] = fs.values
            for mode, eps, kw in (("static", 1e-14, {}), ("static", 0.1, {}),
                                  ("dynamic", 0.1, {}), ("fixed_rank", None, {"fixed_ranks": 2})):
                tt, rep = sparsett.fasttt(t, eps=eps, pivot=p, mode=mode, **kw)
                tag = f"t{i}_p{p}_{mode}_{eps}"
                for k, c in enumerate(tt.cores):
                    arrays[f"{tag}_core{k}"] = np.array(c)
                case["runs"].append({
                    "tag": tag, "pivot": p, "mode": mode, "eps": eps, "kw": kw,
                    "ranks": list(rep.ranks), "ranks_lossless": list(rep.ranks_lossless),
                    "num_fibers": rep.num_fibers, "eps_actual": rep.eps_actual,
                    "eps_actual_method": rep.eps_actual_method,
                    "eps_actual_inner": rep.eps_actual_inner,
                    "flops_fasttt_model": rep.flops_fasttt_model,
                    "flops_ttsvd_model": rep.flops_ttsvd_model,
                })
        cases.append(case)
    # d = 1: the reference's FiberSet rejects its own single-fiber output
    # (tensor.py:326-329 computes r = 0 for an empty fixed tuple), so fasttt
    # raises ValueError; record that behaviour for the drop-in.
    t1 = rand_sparse(rng, (7,), 0.5)
    try:
        sparsett.fasttt(t1)
        d1 = "ok"
    except ValueError as e:
        d1 = "ValueError: " + str(e)
    arrays["d1_coords"] = t1.coords
    arrays["d1_values"] = t1.values
    cases.append({"id": "d1", "shape": [7], "fasttt": d1})
    np.savez_compressed(os.path.join(HERE, "small.npz"), **arrays)
    with open(os.path.join(HERE, "small.json"), "w") as fh:
        json.dump(cases, fh, indent=1)
    print("small", len(cases), "tensors", flush=True)


if __name__ == "__main__":
    for arg in sys.argv[1:] or ["small", "c1", "c2", "c4"]:
        if arg == "c5idx":
            config5_index()
            continue
        if arg == "small":
            small()
        else:
            config(int(arg.lstrip("c")))
