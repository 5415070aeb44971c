"""GPU timeline of one warm decomposition from torch.profiler (CUPTI
activity records; no nsys in the image): busy vs idle time on the stream and
the largest idle gaps with the kernels around them (debug aid).

usage: python tools/timeline.py [config] [ngaps]
"""
import re
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ngaps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)
cd, vd = a.device_arrays()


def step():
    return ft.fasttt_device(a, cd, vd, e, None, "static", None, False, 1.0, report=True)


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()
def short(name):
    m = re.search(r"(k_\w+(<[^>(]*>)?)", name)
    return m.group(1) if m else name.split(" (")[0]


ev = []
api = []
for x in prof.events():
    if x.device_type == torch.autograd.DeviceType.CUDA:
        ev.append((x.time_range.start, x.time_range.end, short(x.name)))
    elif x.name.startswith("cuda") or x.name.startswith("cu"):
        api.append((x.time_range.start, x.time_range.end, x.name))
api.sort()
ev.sort()
t0, t1 = ev[0][0], max(x[1] for x in ev)
busy = 0.0
gaps = []
cur = t0
prev = None
for i, (st, en, name) in enumerate(ev):
    if st > cur:
        gaps.append((st - cur, f"#{i - 1} " + str(prev), name))
    busy += max(0.0, en - max(st, cur))
    cur = max(cur, en)
    prev = name
span = t1 - t0
print(f"config {cfg}: {len(ev)} device activities, span {span / 1e3:.3f} ms, busy {busy / 1e3:.3f} ms, "
      f"idle {(span - busy) / 1e3:.3f} ms")
gaps.sort(reverse=True)
gap_at = {}
cur = t0
for i, (st, en, name) in enumerate(ev):
    if st > cur:
        gap_at[(cur, st)] = st - cur
    cur = max(cur, en)
for (a, b), g in sorted(gap_at.items(), key=lambda x: -x[1])[:ngaps]:
    inside = [(x[2], round(x[1] - x[0], 1)) for x in api if x[0] < b and x[1] > a]
    agg = {}
    for nm, dt in inside:
        agg[nm] = agg.get(nm, 0.0) + dt
    top = sorted(agg.items(), key=lambda x: -x[1])[:4]
    print(f"  gap {g:8.1f} us  runtime calls inside: {len(inside)}  top {top}")
if "--gapdetail" in sys.argv:
    for (a, b), g in sorted(gap_at.items(), key=lambda x: -x[1])[3:7]:
        print(f"  -- gap {g:.1f} us: host API calls from 15 us before its start to its end")
        for x in api:
            if x[1] > a - 15 and x[0] < b:
                print(f"     t={x[0] - a:8.1f} dur={x[1] - x[0]:7.1f}  {x[2]}")
for g, p, n in gaps[:ngaps]:
    print(f"  gap {g:8.1f} us  after {str(p)[:60]:60s} before {str(n)[:60]}")
by = {}
for st, en, name in ev:
    k = name
    by[k] = by.get(k, 0.0) + (en - st)
if "--seq" in sys.argv:
    for i, (st, en, name) in enumerate(ev):
        print(f"  #{i:3d} t={(st - t0):8.1f} dur={en - st:7.1f}  {name}")
print("busy by kernel:")
for k, t in sorted(by.items(), key=lambda x: -x[1])[:25]:
    print(f"  {t:9.1f} us  {k}")
