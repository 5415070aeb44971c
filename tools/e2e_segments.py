"""Host wall time of the public fasttt() call split into its Python-visible
segments (upload calls, the fused native call, the D2H of the slab) on
config 5 (debug aid).

usage: python tools/e2e_segments.py
"""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1908_02721_b200 as ft
from paper_1908_02721_b200 import generators as G, pipeline as P, coo as C
s, c, v, e = G.gen_config(5)
a = ft.SparseTensor(s, c, v)
T = {}
def wrap(mod, name):
    f = getattr(mod, name)
    def g(*x, **k):
        t0 = time.perf_counter(); r = f(*x, **k); T.setdefault(name, []).append((time.perf_counter() - t0) * 1e3); return r
    setattr(mod, name, g)
wrap(P, "_fasttt_fused"); wrap(P, "_slab_to_host")
up = C.SparseTensor._upload
def up2(self):
    t0 = time.perf_counter(); r = up(self); T.setdefault("_upload", []).append((time.perf_counter() - t0) * 1e3); return r
C.SparseTensor._upload = up2
for i in range(8):
    a.drop_device_copy(); torch.cuda.synchronize()
    t0 = time.perf_counter(); ft.fasttt(a, eps=e); T.setdefault("fasttt", []).append((time.perf_counter() - t0) * 1e3)
for k, v in T.items(): print(k, " ".join(f"{x:7.3f}" for x in v[3:]))
