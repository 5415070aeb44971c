import json
import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name):
    """(meta, arrays) for a committed golden fixture, or None if absent."""
    jp = os.path.join(GOLDEN, f"{name}.json")
    zp = os.path.join(GOLDEN, f"{name}.npz")
    if not (os.path.exists(jp) and os.path.exists(zp)):
        return None
    with open(jp) as fh:
        meta = json.load(fh)
    return meta, np.load(zp)


def rand_coo(rng, shape, density):
    """Seeded distinct coordinates + nonzero values (the reference conftest's
    rand_sparse recipe, as raw arrays)."""
    size = math.prod(shape)
    nnz = int(density * size)
    lin = np.sort(rng.permutation(size)[:nnz].astype(np.int64))
    vals = rng.uniform(-1.0, 1.0, nnz)
    vals[vals == 0.0] = 0.5
    coords = np.empty((nnz, len(shape)), dtype=np.int64)
    rem = lin.copy()
    for k in range(len(shape) - 1, -1, -1):
        coords[:, k] = rem % shape[k]
        rem //= shape[k]
    return coords, vals


@pytest.fixture
def rng():
    return np.random.default_rng(1729)
