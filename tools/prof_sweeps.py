"""Host cost of the index sweeps (debug aid): cProfile + per-call timing."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402
from paper_1908_02721_b200 import pipeline as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)
cd, vd = a.device_arrays()
pivot = P.select_p(a)
df = ft.coo.fibers_device(a.shape, pivot, cd, vd, a.nnz)
for _ in range(3):
    P.index_sweeps_device(df)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    P.index_sweeps_device(df)
torch.cuda.synchronize()
print(f"sweeps wall {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    P.index_sweeps_device(df)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
t0 = time.perf_counter()
for _ in range(20):
    ft.coo.fibers_device(a.shape, pivot, cd, vd, a.nnz)
torch.cuda.synchronize()
print(f"fibers wall {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    ft.coo.fibers_device(a.shape, pivot, cd, vd, a.nnz)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
