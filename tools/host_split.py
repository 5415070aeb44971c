"""Split one warm decomposition's host time into time inside native C-ABI
calls (launch + blocked syncs) and Python time around them (debug aid).

usage: python tools/host_split.py [config]
"""
import collections
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import _native as nat  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)
cd, vd = a.device_arrays()
real = nat.load_library()
acc = collections.defaultdict(lambda: [0, 0.0])


class Proxy:
    def __getattr__(self, name):
        fn = getattr(real, name)

        def wrapped(*args):
            t0 = time.perf_counter()
            r = fn(*args)
            acc[name][0] += 1
            acc[name][1] += time.perf_counter() - t0
            return r
        return wrapped


def step():
    return ft.fasttt_device(a, cd, vd, e, None, "static", None, False, 1.0, report=True)


for _ in range(3):
    step()
torch.cuda.synchronize()
nat.lib = lambda: Proxy()
nat.load_library = lambda *x: Proxy()
N = 10
acc.clear()
t0 = time.perf_counter()
for _ in range(N):
    step()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / N * 1e3
cms = sum(x[1] for x in acc.values()) / N * 1e3
print(f"config {cfg}: wall {wall:.3f} ms/decomp, inside native calls {cms:.3f} ms, "
      f"python {wall - cms:.3f} ms, native calls {sum(x[0] for x in acc.values()) / N:.0f}")
for k, (n, t) in sorted(acc.items(), key=lambda x: -x[1][1])[:15]:
    print(f"  {t / N * 1e3:7.3f} ms {n / N:5.1f}x {k}")
