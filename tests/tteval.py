"""Test-side TT evaluator (the checker, not the product): entries of a train
given as numpy cores at integer coordinates, with the math of tt_entry
(reference ttformat.py:110-121) -- the left row vector times one core slice
per mode -- written with plain torch fp64 ops on cuda:0: the points are
grouped by their index in each mode so every step is one dense matmul per
index value (the oracle's grouping, oracle/fasttt_oracle.py tt_entries).
Independent of libfasttt_b200's tt_entries kernels, so it checks them and
the trains they evaluate."""

import numpy as np
import torch


def tt_entries_torch(cores, coords, chunk=1 << 20, device="cuda"):
    coords = np.ascontiguousarray(coords, dtype=np.int64)
    n = coords.shape[0]
    cs = [torch.from_numpy(np.ascontiguousarray(c, dtype=np.float64)).to(device) for c in cores]
    out = np.empty(n)
    for s in range(0, n, chunk):
        idx = torch.from_numpy(coords[s:s + chunk]).to(device)
        b = idx.shape[0]
        v = cs[0][0][idx[:, 0]]  # (b, r1)
        for k in range(1, len(cs)):
            c = cs[k]
            nxt = torch.empty((b, c.shape[2]), dtype=torch.float64, device=device)
            col = idx[:, k]
            for i in range(c.shape[1]):
                rows = torch.nonzero(col == i).squeeze(1)
                if rows.numel():
                    nxt[rows] = v[rows] @ c[:, i, :]
            v = nxt
        out[s:s + chunk] = v[:, 0].cpu().numpy()
    return out
