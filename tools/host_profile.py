"""Host-side cost of one warm decomposition: wall time vs device time, and a
cProfile of the Python/ctypes driver.

usage: python tools/host_profile.py <config> [top_n]
"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)
cd, vd = a.device_arrays()


def step():
    return ft.fasttt_device(a, cd, vd, e, None, "static", None, False, 1.0, report=True)


for _ in range(3):
    step()
torch.cuda.synchronize()
walls, devs = [], []
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    step()
    e1.record()
    torch.cuda.synchronize()
    walls.append((time.perf_counter() - t0) * 1e3)
    devs.append(e0.elapsed_time(e1))
print(f"wall ms {[round(x, 3) for x in walls]}\ndevice ms {[round(x, 3) for x in devs]}")
from paper_1908_02721_b200 import _native as nat  # noqa: E402

lib, ctx = nat.lib(), nat.context()


def stats():
    n = nat.ctypes.c_int64(0)
    w = nat.ctypes.c_double(0)
    lib.ftt_sync_stats(ctx, nat.ctypes.byref(n), nat.ctypes.byref(w))
    return n.value, w.value, nat.kernel_launches()


s0 = stats()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    step()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3 / 5
s1 = stats()
print(f"per step: wall {wall:.3f} ms, native round trips {(s1[0] - s0[0]) / 5:.1f}, "
      f"blocked {(s1[1] - s0[1]) / 5:.3f} ms, launches {(s1[2] - s0[2]) / 5:.1f}")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(top)
st.sort_stats("cumulative").print_stats(top)
