"""Host time between consecutive native calls of one warm decomposition
(debug aid): the Python (or C++ host) work the GPU waits for when the stream
runs dry.

usage: python tools/host_gaps.py [config] [top]
"""
import sys
import time
import traceback

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import _native as nat  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)
cd, vd = a.device_arrays()
real = nat.load_library()
log = []


class Proxy:
    def __getattr__(self, name):
        fn = getattr(real, name)

        def wrapped(*args):
            t0 = time.perf_counter()
            r = fn(*args)
            t1 = time.perf_counter()
            where = traceback.extract_stack(limit=3)[0]
            log.append((t0, t1, name, f"{where.filename.split('/')[-1]}:{where.lineno}"))
            return r
        return wrapped


def step():
    return ft.fasttt_device(a, cd, vd, e, None, "static", None, False, 1.0, report=True)


for _ in range(3):
    step()
torch.cuda.synchronize()
nat.lib = lambda: Proxy()
nat.load_library = lambda *x: Proxy()
import gc
gc.collect()
gc.disable()
log.clear()
t_start = time.perf_counter()
step()
t_end = time.perf_counter()
gaps = []
for (a0, a1, n0, w0), (b0, b1, n1, w1) in zip(log, log[1:]):
    gaps.append((b0 - a1, n0, n1, w1))
inside = sum(x[1] - x[0] for x in log)
print(f"config {cfg}: wall {1e3 * (t_end - t_start):.3f} ms, native calls {len(log)}, inside "
      f"{1e3 * inside:.3f} ms, between {1e3 * sum(g[0] for g in gaps):.3f} ms")
for g, n0, n1, w in sorted(gaps, reverse=True)[:top]:
    print(f"  {1e6 * g:8.1f} us  after {n0:28s} before {n1:28s} ({w})")
