"""Split the public fasttt() call (host buffers in, host cores out) into its
phases: H2D staging + device COO rebuild, the device decomposition, and the
D2H of the cores (debug aid for the e2e leg of bench.py).

usage: python tools/e2e_split.py [config] [reps]
"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402
from paper_1908_02721_b200 import pipeline as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)


def now():
    torch.cuda.synchronize()
    return time.perf_counter()


for i in range(reps + 2):
    a.drop_device_copy()
    t0 = now()
    cd, vd = a.device_arrays()
    t1 = now()
    res = P.fasttt_device(a, cd, vd, e, None, "static", None, False, 1.0, report=True)
    t2 = now()
    host = P._cores_to_host(res.cores)
    t3 = now()
    a.drop_device_copy()
    del cd, vd
    t4 = now()
    tt, rep = ft.fasttt(a, eps=e)
    t5 = now()
    print(f"rep {i}: h2d+rebuild {1e3 * (t1 - t0):8.3f}  device {1e3 * (t2 - t1):8.3f}  "
          f"d2h {1e3 * (t3 - t2):8.3f}  | fasttt() {1e3 * (t5 - t4):8.3f} ms", flush=True)
print("memory allocated %.2f GB reserved %.2f GB" % (torch.cuda.memory_allocated() / 1e9,
                                                     torch.cuda.memory_reserved() / 1e9))
