"""Stream-ordered pool state around warm decompositions (debug aid): the
device's default / current memory pools, their release threshold and
reserved / used bytes, and the wall time of each decomposition.

usage: python tools/pool_probe.py [config] [reps]
"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
s, c, v, e = G.gen_config(cfg)
a = ft.SparseTensor(s, c, v)
cd, vd = a.device_arrays()


def pool_state(tag):
    _, dpool = rt.cudaDeviceGetDefaultMemPool(0)
    _, cpool = rt.cudaDeviceGetMemPool(0)
    out = []
    for name, pool in (("default", dpool), ("current", cpool)):
        vals = []
        for attr in ("cudaMemPoolAttrReleaseThreshold", "cudaMemPoolAttrReservedMemCurrent",
                     "cudaMemPoolAttrUsedMemCurrent", "cudaMemPoolAttrReservedMemHigh"):
            err, val = rt.cudaMemPoolGetAttribute(pool, getattr(rt.cudaMemPoolAttr, attr))
            vals.append(int(val) if not err else f"err{int(err)}")
        out.append(f"{name}={int(pool)} thr={vals[0]} reserved={vals[1]} used={vals[2]} high={vals[3]}")
    print(tag, " | ".join(out), flush=True)


pool_state("before")
for i in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ft.fasttt_device(a, cd, vd, e, None, "static", None, False, 1.0, report=True)
    torch.cuda.synchronize()
    print(f"rep {i}: {1e3 * (time.perf_counter() - t0):.3f} ms", flush=True)
    pool_state(f"after {i}")
