"""Device time of one A3 resolve launch (k_resolve core) on adjacency
matrices shaped like the workloads' first tiles (BM_RESOLVE_BENCH=1)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ["BM_RESOLVE_BENCH"] = "1"
from paper_2601_01405_b200 import bm as B  # noqa: E402
from workloads import gen  # noqa: E402


def adjacency(X, eps2):
    nc = len(X)
    D = ((X[:, None, :].astype(np.float64) - X[None, :, :]) ** 2).sum(-1)
    A = np.tril(D < eps2, -1)
    W = (nc + 31) // 32
    out = np.zeros((nc, W), dtype=np.uint32)
    for a in range(nc):
        for b in np.nonzero(A[a])[0]:
            out[a, b >> 5] |= np.uint32(1) << np.uint32(b & 31)
    return out


for name in ("c2", "c3_e8", "c4"):
    w = gen.get(name)
    X = gen.generate(w, 1024)
    eps2 = w.eps ** 2
    adj = adjacency(X.astype(np.float64), eps2)
    lm = B.resolve_tile(adj, 1024)
    print(name, "landmarks in tile", int(lm.sum()), flush=True)
adj0 = np.zeros((1024, 32), dtype=np.uint32)
B.resolve_tile(adj0, 1024)
B.resolve_tile(adj0, 64)
