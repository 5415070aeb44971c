"""Input side: COO text and MatrixMarket readers.
Host-only (no GPU): the native fast path against the reference's line loop
(formats.py:47-127), error texts, bit-exact round trips."""
import os
import warnings

import numpy as np
import pytest
import scipy.io
import scipy.sparse as sp

import paper_1908_02721_b200 as ft
from paper_1908_02721_b200 import formats as F


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


@pytest.mark.parametrize("shape,density,seed", [((4, 5, 6), 0.3, 1), ((9, 2, 3, 7), 0.1, 2),
                                                ((50,), 0.5, 3), ((3, 3), 1.0, 4)])
def test_coo_round_trip_bit_exact(tmp_path, shape, density, seed):
    rng = np.random.default_rng(seed)
    size = int(np.prod(shape))
    lin = np.sort(rng.permutation(size)[: max(1, int(density * size))])
    coords = np.stack(np.unravel_index(lin, shape), 1)
    vals = rng.standard_normal(lin.size) * 10.0 ** rng.integers(-300, 300, lin.size)
    t = ft.SparseTensor(shape, coords, vals)
    p = str(tmp_path / "t.coo")
    ft.write_coo(t, p)
    assert F._native_parse(p) is not None  # the native path read it
    u = ft.ingest_coo(p)
    assert u.shape == t.shape
    assert np.array_equal(u.coords, t.coords) and np.array_equal(u.values, t.values)
    r = F._ingest_coo_reference(p)
    assert np.array_equal(r.coords, u.coords) and np.array_equal(r.values, u.values)


def test_coo_native_handles_layout_variants(tmp_path):
    text = "# shape 3 4\n\n  1 2   0.5\r\n3 4 -2e-3\n\t2 1 +7\n"
    p = _write(tmp_path, "v.coo", text)
    fast = F._native_parse(p)
    assert fast is not None
    u, r = ft.ingest_coo(p), F._ingest_coo_reference(p)
    assert np.array_equal(u.coords, r.coords) and np.array_equal(u.values, r.values)


@pytest.mark.parametrize("text,msg", [
    ("", "empty file, missing shape header"),
    ("#shape 3 3\n1 1 1.0\n", ":1: expected header"),
    ("# shape 3 0\n", ":1: bad shape header"),
    ("# shape 3 3\n1 1\n", ":2: expected 2 indices and a value, got 2 fields"),
    ("# shape 3 3\n1 1 1.0\n2 x 1.0\n", ":3: unparsable entry"),
    ("# shape 3 3\n4 1 1.0\n", ":2: index 4 out of range 1..3 in mode 1"),
    ("# shape 3 3\n1 0 1.0\n", ":2: index 0 out of range 1..3 in mode 2"),
    ("# shape 3 3\n1 1 nan\n", ":2: non-finite value nan"),
    ("# shape 3 3\n1 1 1.0\n1 1 2.0\n", "duplicate coordinate"),
    ("# shape 3 3\n1 1 0x10\n", ":2: unparsable entry"),
])
def test_coo_errors_match_reference_text(tmp_path, text, msg):
    p = _write(tmp_path, "bad.coo", text)
    with pytest.raises(ft.FormatError) as e:
        ft.ingest_coo(p)
    assert msg in str(e.value)


def test_coo_python_literal_forms_fall_back(tmp_path):
    # forms Python's int()/float() accept and strtoll/strtod do not
    p = _write(tmp_path, "u.coo", "# shape 20 3\n1_0 1 1_0.5\n2 2 1e-1\n")
    assert F._native_parse(p) is None
    t = ft.ingest_coo(p)
    assert t.coords.tolist() == [[1, 1], [9, 0]] and t.values.tolist() == [0.1, 10.5]


def test_coo_no_entries_warns(tmp_path):
    p = _write(tmp_path, "z.coo", "# shape 2 2\n\n")
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        t = ft.ingest_coo(p)
    assert t.nnz == 0 and t.shape == (2, 2)
    assert any("no entries" in str(x.message) for x in w)


def test_matrix_market_general_and_symmetric(tmp_path):
    rng = np.random.default_rng(8)
    a = sp.random(30, 20, density=0.2, random_state=rng, format="coo")
    p = str(tmp_path / "g.mtx")
    scipy.io.mmwrite(p, a)
    m = ft.ingest_matrix_market(p)
    assert np.array_equal(m.toarray(), a.toarray())
    s = sp.random(25, 25, density=0.2, random_state=rng)
    s = (s + s.T).tocoo()
    p2 = str(tmp_path / "s.mtx")
    scipy.io.mmwrite(p2, s, symmetry="symmetric")
    assert np.allclose(ft.ingest_matrix_market(p2).toarray(), s.toarray())
    bad = _write(tmp_path, "b.mtx", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n")
    with pytest.raises(ft.FormatError, match="unsupported MatrixMarket format 'array'"):
        ft.ingest_matrix_market(bad)
    cpx = _write(tmp_path, "c.mtx", "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n")
    with pytest.raises(ft.FormatError, match="field 'complex'"):
        ft.ingest_matrix_market(cpx)
    assert os.path.exists(p)
