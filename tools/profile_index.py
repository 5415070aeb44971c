"""One warm index pass (select_p counts, fiber extraction, deparallelisation
sweeps) on the device COO bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` captures of the sort/segment kernels.

usage: python tools/profile_index.py [config]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402
from paper_1908_02721_b200 import pipeline as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)
cd, vd = a.device_arrays()
pivot = P.select_p(a)


def once():
    P._fiber_counts_device(a)
    df = ft.coo.fibers_device(a.shape, pivot, cd, vd, a.nnz, lin_d=a.device_lin())
    return P.index_sweeps_device(df)


for _ in range(2):
    once()
torch.cuda.synchronize()
torch.cuda.profiler.start()
once()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
