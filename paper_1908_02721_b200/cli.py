"""``python -m paper_1908_02721_b200 decompose --in X --device cuda:0`` -- the
``--device`` row of SURVEY.md 8(f3): the reference's ``decompose`` command
(cli.py:122-144, 259-271) for ``--method fasttt`` on one B200.

Only the hot path's front door: the same input flags, summary lines and exit
codes (0 within budget, 1 error contract missed / contract violation, 2
unusable input; cli.py:300-315).  The JSON report schema, ``.npz`` archives,
``--method ttsvd``, ``bench`` and the generators are out of scope (DESIGN 8).
"""

from __future__ import annotations

import argparse
import math
import sys
from pathlib import Path

from .coo import ContractViolationError, FormatError
from .formats import ingest_coo, ingest_matrix_market

__all__ = ["main"]


def _int_tuple(text):
    try:
        return tuple(int(tok) for tok in str(text).replace(",", " ").split())
    except ValueError:
        raise FormatError(f"expected comma-separated integers, got {text!r}") from None


def _select_device(spec: str) -> None:
    """``cuda`` or ``cuda:N``; anything else (the reference has only the CPU)
    is refused -- there is no CPU path behind this command."""
    import torch

    name, _, idx = spec.partition(":")
    if name != "cuda" or (idx and not idx.isdigit()):
        raise FormatError(f"--device expects cuda or cuda:N, got {spec!r}")
    if not torch.cuda.is_available():
        raise OSError("--device: no CUDA device is visible")
    n = int(idx) if idx else 0
    if n >= torch.cuda.device_count():
        raise FormatError(f"--device cuda:{n}: only {torch.cuda.device_count()} device(s) visible")
    torch.cuda.set_device(n)


def _load_input(path, row_dims, col_dims):
    from .trains import tensorize_matrix

    if Path(path).suffix.lower() in (".mtx", ".mm"):
        if row_dims is None or col_dims is None:
            raise FormatError(f"{path}: matrix input needs --row-dims and --col-dims")
        rd, cd = _int_tuple(row_dims), _int_tuple(col_dims)
        # fused, sorted and coalesced on the GPU; the COO stays resident
        return tensorize_matrix(ingest_matrix_market(path), rd, cd, device=True)
    return ingest_coo(path)


def cmd_decompose(args) -> int:
    from .pipeline import fasttt

    _select_device(args.device)
    tensor = _load_input(args.input, args.row_dims, args.col_dims)
    eps = args.eps if args.eps is not None else 1e-14
    mode = "fixed_rank" if args.mode == "fixed" else args.mode
    ranks = _int_tuple(args.ranks) if args.ranks else None
    if mode == "fixed_rank" and ranks is None:
        raise FormatError("--mode fixed needs --ranks")
    if ranks is not None and len(ranks) == 1:
        ranks = ranks[0]
    pivot = args.p - 1 if args.p is not None else None
    _, rep = fasttt(tensor, eps=eps, pivot=pivot, mode=mode, fixed_ranks=ranks)
    for note in rep.warnings:
        print(f"warning: {note}", file=sys.stderr)
    sigma = rep.nnz / math.prod(rep.shape) if rep.shape else 0.0
    print("method       fasttt")
    print(f"shape        {tuple(rep.shape)}  nnz {rep.nnz}  sigma {sigma:.3e}")
    print(f"pivot p      {rep.pivot + 1}   fibers R {rep.num_fibers}")
    print(f"r_tilde      {list(rep.ranks_lossless)}")
    print(f"r            {list(rep.ranks)}")
    print(f"eps          {rep.eps:.3e}   eps_actual {rep.eps_actual:.3e}")
    print(f"wall_time_s  {rep.wall_time_s:.6f}   device {args.device}")
    if args.mode == "fixed" and args.eps is None:
        return 0  # no error contract was requested
    return 0 if rep.eps_actual <= eps + 1e-12 else 1


def _build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="paper_1908_02721_b200",
        description="FastTT decomposition of a sparse tensor or matrix on one B200.",
    )
    sub = parser.add_subparsers(dest="command", required=True)
    dec = sub.add_parser("decompose", help="decompose one tensor or matrix")
    dec.add_argument("--in", dest="input", required=True, help=".coo or .mtx input")
    dec.add_argument("--method", choices=("fasttt",), default="fasttt")
    dec.add_argument("--eps", type=float, default=None, help="relative error budget (default 1e-14)")
    dec.add_argument("--p", type=int, default=None, help="pivot mode, 1-based (default: auto)")
    dec.add_argument("--mode", choices=("static", "dynamic", "fixed"), default="static")
    dec.add_argument("--ranks", default=None, help="interior rank targets for --mode fixed")
    dec.add_argument("--row-dims", default=None, help="row factorization for matrix input")
    dec.add_argument("--col-dims", default=None, help="column factorization for matrix input")
    dec.add_argument("--device", default="cuda:0", help="cuda or cuda:N (default cuda:0)")
    dec.set_defaults(func=cmd_decompose)
    return parser


def main(argv=None) -> int:
    args = _build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (FormatError, OSError, ValueError, TypeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except ContractViolationError as exc:
        print(f"contract violation: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
