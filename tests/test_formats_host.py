"""Input side: COO text and MatrixMarket readers.
Host-only (no GPU): the native fast path against the reference's line loop
(formats.py:47-127), error texts, bit-exact round trips."""
import json
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


CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "coo_cases.json")))


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
    u = ft.ingest_coo(p)
    assert u.shape == t.shape
    assert np.array_equal(u.coords, t.coords) and np.array_equal(u.values, t.values)


@pytest.mark.parametrize("case", range(len(CASES)))
def test_coo_reader_matches_reference(tmp_path, case):
    """Every committed case (tests/golden/make_golden.py coo_cases: the
    unmodified reference's ingest_coo on well-formed and malformed texts):
    the same tensor bit for bit, or the same exception type and message."""
    rec = CASES[case]
    p = tmp_path / "case.coo"
    p.write_bytes(rec["text"].encode("ascii"))
    if rec["ok"]:
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            t = ft.ingest_coo(str(p))
        assert list(t.shape) == rec["shape"]
        assert t.coords.tolist() == rec["coords"]
        assert [float.hex(float(v)) for v in t.values] == rec["values"]
        assert [str(x.message).replace(str(p), "{path}") for x in w] == rec["warnings"]
    else:
        with pytest.raises(Exception) as e:
            ft.ingest_coo(str(p))
        assert type(e.value).__name__ == rec["type"]
        assert str(e.value).replace(str(p), "{path}") == rec["message"]


def test_coo_reader_rejects_non_ascii(tmp_path):
    p = tmp_path / "u.coo"
    p.write_bytes(b"# shape 3 3\n1 1 1.0\n2 2 \xc3\xa9\n")
    with pytest.raises(UnicodeDecodeError):
        ft.ingest_coo(str(p))


def test_coo_reader_random_lines_match_python_literals(tmp_path):
    """Fuzz: tokens built from the characters of Python literals; the native
    grammar accepts exactly what int()/float() accept, with the same value."""
    rng = np.random.default_rng(11)
    alphabet = list("0123456789_+-.eEinfaINFA ")
    for trial in range(300):
        tok = "".join(rng.choice(alphabet, int(rng.integers(1, 8)))).strip() or "1"
        if " " in tok:
            continue
        p = tmp_path / f"f{trial}.coo"
        p.write_text(f"# shape 9 9\n1 2 {tok}\n")
        try:
            want = float(tok)
        except ValueError:
            want = None
        if want is None:
            with pytest.raises(ft.FormatError, match="unparsable entry"):
                ft.ingest_coo(str(p))
        elif not np.isfinite(want):
            with pytest.raises(ft.FormatError, match="non-finite value"):
                ft.ingest_coo(str(p))
        else:
            t = ft.ingest_coo(str(p))
            got = t.values.tolist()
            assert got == ([want] if want != 0.0 else []), tok


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


def test_matrix_market_native_body_equals_scipy(tmp_path):
    """The strict native body reader gives scipy.io.mmread's arrays in its
    order (symmetric: stored entries, then mirrored off-diagonal ones);
    bodies outside the strict grammar go to scipy for its result or error."""
    sym = ("%%MatrixMarket matrix coordinate real symmetric\n% c\n4 4 5\n1 1 1.5\n3 1 2.0\n"
           "4 2 3e0\n2 2 -1\n4 3 7\n")
    gen = "%%MatrixMarket matrix coordinate real general\n3 3 4\n1 1 1.5\n3 1 2.0\n1 1 3\n2 2 -1\n"
    for name, text in (("s.mtx", sym), ("g.mtx", gen)):
        p = _write(tmp_path, name, text)
        m = ft.ingest_matrix_market(p)
        ref = sp.coo_matrix(scipy.io.mmread(p), dtype=np.float64)
        assert m.shape == ref.shape
        assert m.row.tolist() == ref.row.tolist() and m.col.tolist() == ref.col.tolist()
        assert m.data.tolist() == ref.data.tolist()
    short = _write(tmp_path, "t.mtx", "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1\n")
    with pytest.raises(ft.FormatError, match="Truncated file"):
        ft.ingest_matrix_market(short)
    oob = _write(tmp_path, "o.mtx", "%%MatrixMarket matrix coordinate real general\n3 3 1\n4 1 1\n")
    with pytest.raises(ft.FormatError, match="out of bounds"):
        ft.ingest_matrix_market(oob)
    with pytest.raises(ft.FormatError, match="not a MatrixMarket file"):
        ft.ingest_matrix_market(_write(tmp_path, "n.mtx", "hello\n"))
    with pytest.raises(ft.FormatError, match="symmetry 'hermitian'"):
        ft.ingest_matrix_market(_write(
            tmp_path, "h.mtx", "%%MatrixMarket matrix coordinate real Hermitian\n1 1 1\n1 1 1\n"))
