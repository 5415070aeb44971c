"""Debug timing of whole decompositions per config (FTT_DEBUG=1 prints per-SVD stats)."""
import sys
import time

sys.path.insert(0, ".")
import paper_1908_02721_b200 as ft  # noqa: E402
from paper_1908_02721_b200 import generators as G  # noqa: E402

for cfg in [int(x) for x in sys.argv[1].split(",")]:
    s, c, v, e = G.gen_config(cfg)
    a = ft.SparseTensor(s, c, v)
    t0 = time.time()
    tt, rep = ft.fasttt(a, eps=e)
    print("cfg", cfg, f"{time.time() - t0:.3f}s", rep.pivot, rep.ranks, file=sys.stderr, flush=True)
