"""cProfile of warm public fasttt() calls with a fresh upload each (host-side
Python cost of the e2e path; debug aid).

usage: python tools/py_profile_e2e.py [config] [reps]
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
for _ in range(3):
    a.drop_device_copy()
    ft.fasttt(a, eps=e)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(reps):
    a.drop_device_copy()
    ft.fasttt(a, eps=e)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(22)
