"""One warm fasttt decomposition bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists and captures.

usage: python tools/profile_step.py <config> [device|e2e]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)
cd, vd = a.device_arrays()
for _ in range(2):
    ft.fasttt_device(a, cd, vd, e, None, "static", None, False, 1.0, report=True)
torch.cuda.synchronize()
torch.cuda.profiler.start()
res = ft.fasttt_device(a, cd, vd, e, None, "static", None, False, 1.0, report=True)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ranks", res.ranks, file=sys.stderr)
