"""CUPTI timeline of one warm public fasttt() call (host buffers in, host
cores out): the first device activities with their start times, to see how
the H2D of the COO overlaps the first kernels (debug aid).

usage: python tools/timeline_e2e.py [config] [n]
"""
import re
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)
for _ in range(3):
    a.drop_device_copy()
    ft.fasttt(a, eps=e)
torch.cuda.synchronize()
a.drop_device_copy()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    ft.fasttt(a, eps=e)
    torch.cuda.synchronize()
ev = []
for x in prof.events():
    if x.device_type == torch.autograd.DeviceType.CUDA:
        m = re.search(r"(k_\w+(<[^>(]*>)?)", x.name)
        ev.append((x.time_range.start, x.time_range.end, m.group(1) if m else x.name.split(" (")[0]))
ev.sort()
t0 = ev[0][0]
print(f"config {cfg}: {len(ev)} device activities, span {(max(x[1] for x in ev) - t0) / 1e3:.3f} ms")
for st, en, name in ev[:n]:
    print(f"  t={st - t0:9.1f} dur={en - st:8.1f}  {name}")
