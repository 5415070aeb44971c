"""Latency of the narrow direct SVD (k_jacobi_qr path) on short tall
operands like config 5's B^T (512 x 16, 130 x 16): device us per call
(CUDA events, warm), for a Gaussian and a graded spectrum.

usage: python tools/jqr_probe.py [reps]
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_02721_b200 import dense  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(0)
for m, n in ((512, 16), (130, 16), (430, 16)):
    for kind in ("gauss", "graded"):
        if kind == "gauss":
            A = rng.standard_normal((m, n))
        else:
            u, _ = np.linalg.qr(rng.standard_normal((m, n)))
            v, _ = np.linalg.qr(rng.standard_normal((n, n)))
            A = (u * np.logspace(0, -9, n)) @ v.T
        Ad = torch.from_numpy(np.asfortranarray(A).T.copy()).cuda()
        s = dense.dev_svd_values(Ad, m, n, m, False)
        err = np.max(np.abs(s - np.linalg.svd(A, compute_uv=False)) / s[0])
        for _ in range(3):
            dense.dev_svd_values(Ad, m, n, m, False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            dense.dev_svd_values(Ad, m, n, m, False)
        e1.record()
        torch.cuda.synchronize()
        print(f"{m:5d} x {n:2d} {kind:6s} {1e3 * e0.elapsed_time(e1) / reps:8.1f} us/call  "
              f"max rel err {err:.2e}", flush=True)
