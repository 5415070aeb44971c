"""Per-phase host split of one warm decomposition (debug aid): wall time of
each pipeline phase vs the time inside native calls during it."""
import collections
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import _native as nat  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402
from paper_1908_02721_b200 import pipeline as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)
cd, vd = a.device_arrays()
real = nat.load_library()
state = {"native": 0.0}


class Proxy:
    def __getattr__(self, name):
        fn = getattr(real, name)

        def wrapped(*args):
            t0 = time.perf_counter()
            r = fn(*args)
            state["native"] += time.perf_counter() - t0
            return r
        return wrapped


phases = collections.defaultdict(lambda: [0.0, 0.0])


def wrap(mod, name):
    f = getattr(mod, name)

    def w(*args, **kw):
        n0 = state["native"]
        t0 = time.perf_counter()
        r = f(*args, **kw)
        phases[name][0] += time.perf_counter() - t0
        phases[name][1] += state["native"] - n0
        return r
    setattr(mod, name, w)


for name in ("select_p", "fibers_device", "index_sweeps_device", "_structured_train",
             "_sweep_rounding_device", "_inner_error_device"):
    wrap(P, name)


def step():
    return ft.fasttt_device(a, cd, vd, e, None, "static", None, False, 1.0, report=True)


for _ in range(3):
    step()
torch.cuda.synchronize()
nat.lib = lambda: Proxy()
nat.load_library = lambda *x: Proxy()
phases.clear()
N = 10
t0 = time.perf_counter()
for _ in range(N):
    step()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / N * 1e3
print(f"config {cfg}: {wall:.3f} ms per decomposition")
for k, (w, n) in phases.items():
    print(f"  {k:26s} wall {w / N * 1e3:7.3f} ms  native {n / N * 1e3:7.3f} ms  "
          f"python {(w - n) / N * 1e3:7.3f} ms")
