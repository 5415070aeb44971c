"""Micro-benchmarks of the dense kernels (debug aid): DMMA GEMM shapes from
the QR trailing updates, the standalone QR and SVD."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_02721_b200 import _native as nat  # noqa: E402
from paper_1908_02721_b200 import trains as T  # noqa: E402
from paper_1908_02721_b200 import dense as D  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dm = nat.ctypes.c_double(0)
nat.check(nat.lib().ftt_bench_dmma(nat.context(), 20000, nat.ctypes.byref(dm)))
print(f"dmma peak {dm.value:.2f} TFLOP/s", flush=True)
for (ta, tb, m, n, k) in [(0, 0, 314928, 4032, 128), (1, 0, 128, 4032, 314928), (0, 0, 4096, 4096, 4096),
                          (0, 0, 10366, 480, 32), (1, 0, 32, 480, 10366), (0, 0, 25168, 4916, 128)]:
    A = torch.randn((k, m) if not ta else (m, k), dtype=torch.float64, device="cuda")  # col-major m x k == row-major k x m
    B = torch.randn((n, k) if not tb else (k, n), dtype=torch.float64, device="cuda")
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda")
    lda = m if not ta else k
    ldb = k if not tb else n
    ms = timeit(lambda: T.dgemm(ta, tb, m, n, k, 1.0, A, lda, B, ldb, 0.0, C, m))
    print(f"gemm ta={ta} tb={tb} {m}x{n}x{k}: {ms:.3f} ms {2 * m * n * k / ms / 1e9:.2f} TFLOP/s",
          flush=True)
    del A, B, C
for (m, n) in [(10366, 512), (31968, 2282), (25168, 4916), (314928, 4160)]:
    A = torch.randn((n, m), dtype=torch.float64, device="cuda")
    ms = timeit(lambda: T.dev_qr(A, m, n, m), reps=2)
    print(f"qr {m}x{n}: {ms:.2f} ms {(2 * m * n * n - 2 * n ** 3 / 3) / ms / 1e9:.2f} TFLOP/s (R only "
          "counts; Q formation included)", flush=True)
    del A
for (m, n) in [(10366, 512), (4096, 4096)]:
    A = torch.randn((n, m), dtype=torch.float64, device="cuda")
    ms = timeit(lambda: D.dev_svd_values(A, m, n, m, False), reps=1)
    print(f"svd values {m}x{n}: {ms:.2f} ms", flush=True)
