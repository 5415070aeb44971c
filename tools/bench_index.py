"""Index-path stages on one config (device ms per call, CUDA events, warm,
inputs resident): select_p fiber counts, fiber extraction (sort + segment),
the deparallelisation sweeps.  Prints achieved GB/s against the algorithmic
bytes of DESIGN.md section 3.

usage: python tools/bench_index.py [config] [reps]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402
from paper_1908_02721_b200 import pipeline as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)
cd, vd = a.device_arrays()
d, nnz = a.ndim, a.nnz


def timed(fn):
    out = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


ms, counts = timed(lambda: P._fiber_counts_device(a))
pivot = P.select_p(a)
print(f"config {cfg}: nnz {nnz}, d {d}, pivot {pivot}, counts {counts}")
b = nnz * (8 * d + 8) + d * nnz * 16
print(f"select_p counts   {ms:8.3f} ms  {b / ms / 1e6:8.0f} GB/s (alg {b / 1e6:.0f} MB: COO + 16 B/nnz/pivot)")
for _ in range(3):
    ms, df = timed(lambda: ft.coo.fibers_device(a.shape, pivot, cd, vd, nnz))
    print(f"  (extract fibers {ms:.3f} ms)")
b = nnz * (8 * d + 8) + 16 * nnz + 8 * d * df.R
print(f"extract fibers    {ms:8.3f} ms  {b / ms / 1e6:8.0f} GB/s (alg {b / 1e6:.0f} MB), R {df.R}")
ms, sw = timed(lambda: P.index_sweeps_device(df))
kept = sum(int(k.shape[0]) for k, _ in sw.left + sw.right)
b = 8 * df.R * (d - 1) * 2 + 8 * kept
print(f"index sweeps      {ms:8.3f} ms  {b / ms / 1e6:8.0f} GB/s (alg {b / 1e6:.0f} MB)")
