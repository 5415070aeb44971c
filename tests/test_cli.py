"""The ``decompose --device`` front door (reference cli.py:122-144,
259-271, 300-315): flags, summary lines and exit codes 0 / 1 / 2."""
import numpy as np
import pytest

import paper_1908_02721_b200 as ft
from paper_1908_02721_b200 import cli


def _write_case(tmp_path, seed=5):
    rng = np.random.default_rng(seed)
    shape = (6, 5, 7, 4)
    size = int(np.prod(shape))
    lin = np.sort(rng.permutation(size)[: size // 4])
    coords = np.stack(np.unravel_index(lin, shape), 1).astype(np.int64)
    t = ft.SparseTensor(shape, coords, rng.uniform(-1.0, 1.0, lin.size))
    p = tmp_path / "t.coo"
    ft.write_coo(t, p)
    return t, str(p)


def test_parser_defaults_and_flags():
    a = cli._build_parser().parse_args(["decompose", "--in", "x.coo"])
    assert (a.device, a.method, a.mode, a.eps, a.p) == ("cuda:0", "fasttt", "static", None, None)
    a = cli._build_parser().parse_args(
        ["decompose", "--in", "x.mtx", "--device", "cuda:3", "--p", "2", "--mode", "fixed",
         "--ranks", "4,4", "--row-dims", "2,2", "--col-dims", "2,2", "--eps", "1e-6"])
    assert (a.device, a.p, a.mode, a.ranks, a.eps) == ("cuda:3", 2, "fixed", "4,4", 1e-6)
    with pytest.raises(SystemExit):
        cli._build_parser().parse_args(["decompose", "--in", "x.coo", "--method", "ttsvd"])


def test_bad_device_and_input_exit_2(tmp_path, capsys):
    _, path = _write_case(tmp_path)
    assert cli.main(["decompose", "--in", path, "--device", "cpu"]) == 2
    assert "--device expects cuda" in capsys.readouterr().err
    assert cli.main(["decompose", "--in", path, "--device", "cuda:x"]) == 2


@pytest.mark.gpu
def test_decompose_on_device(tmp_path, capsys):
    t, path = _write_case(tmp_path)
    assert cli.main(["decompose", "--in", path, "--eps", "1e-10", "--device", "cuda:0"]) == 0
    out = capsys.readouterr().out
    _, rep = ft.fasttt(t, eps=1e-10)
    assert f"pivot p      {rep.pivot + 1}   fibers R {rep.num_fibers}" in out
    assert f"r_tilde      {list(rep.ranks_lossless)}" in out
    assert f"r            {list(rep.ranks)}" in out
    # 1-based --p, fixed mode without an error contract
    assert cli.main(["decompose", "--in", path, "--p", "2", "--mode", "fixed", "--ranks", "2",
                     "--device", "cuda"]) == 0
    assert "r            [2, 2, 2]" in capsys.readouterr().out
    # a budget the fixed ranks cannot meet: exit 1
    assert cli.main(["decompose", "--in", path, "--mode", "fixed", "--ranks", "1",
                     "--eps", "1e-12"]) == 1
    # unusable input: exit 2
    assert cli.main(["decompose", "--in", str(tmp_path / "missing.coo")]) == 2
    assert cli.main(["decompose", "--in", path, "--mode", "fixed"]) == 2
    m = tmp_path / "m.mtx"
    m.write_text("%%MatrixMarket matrix coordinate real general\n4 4 3\n1 1 1.0\n2 3 -2.0\n4 4 0.5\n")
    assert cli.main(["decompose", "--in", str(m)]) == 2
    assert cli.main(["decompose", "--in", str(m), "--row-dims", "2,2", "--col-dims", "2,2"]) == 0
    assert "shape        (4, 4)  nnz 3" in capsys.readouterr().out
