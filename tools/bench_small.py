"""Latency of the narrow QR / SVD entry points per shape (device ms per call,
CUDA events, warm).

usage: python tools/bench_small.py
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_02721_b200 import trains, dense  # noqa: E402

SHAPES = [(256, 24), (512, 24), (512, 37), (281, 24), (64, 32), (10366, 24), (62206, 32),
          (314928, 32), (4160, 32), (512, 64)]


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


rng = np.random.default_rng(0)
for m, n in SHAPES:
    r = min(8, n)
    A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    Ad = torch.from_numpy(np.asfortranarray(A).T.copy()).cuda()  # column-major m x n
    tq = timed(lambda: trains.dev_qr(Ad, m, n, m))
    ts = timed(lambda: dense.dev_svd_values(Ad, m, n, m, False))
    print(f"{m:7d} x {n:3d}  qr {tq * 1e3:8.1f} us   svd(values) {ts * 1e3:8.1f} us", flush=True)
