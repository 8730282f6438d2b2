import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2601_01405_b200 as bm
d = int(sys.argv[1]) if len(sys.argv) > 1 else 3
zero = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(d)
n = 3000
X = rng.normal(size=(n, d)).astype(np.float32)
if zero:
    X[::97] = 0.0
X[1::5] = X[0::5][: len(X[1::5])] * np.float32(3.0)
eps = 0.05 if d > 3 else 0.02
cov = bm.cover_build(torch.from_numpy(X).cuda(), "cos", eps, path="tensor", tile=256)
print("ok", cov.L, cov.M, cov.E)
