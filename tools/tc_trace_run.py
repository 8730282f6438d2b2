import os, sys
sys.path.insert(0, ".")
import torch
import paper_2601_01405_b200 as bm
from workloads import gen
w = gen.get(sys.argv[1])
X = torch.from_numpy(gen.generate(w)).cuda()
for r in range(3):
    c = bm.cover_build(X, w.metric, w.eps)
    print("L", c.L, file=sys.stderr, flush=True)
    c.free()
