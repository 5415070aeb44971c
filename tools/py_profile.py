"""cProfile of warm device decompositions (host-side Python cost; debug aid).

usage: python tools/py_profile.py [config] [reps]
"""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)
cd, vd = a.device_arrays()
for _ in range(3):
    ft.fasttt_device(a, cd, vd, e, None, "static", None, False, 1.0, report=True)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(reps):
    ft.fasttt_device(a, cd, vd, e, None, "static", None, False, 1.0, report=True)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
