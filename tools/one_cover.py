"""Run N covers of a workload (diagnostics / ncu target): python tools/one_cover.py c3_e8 [N] [tile]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_01405_b200 as bm  # noqa: E402
from workloads import gen  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
tile = int(sys.argv[3]) if len(sys.argv) > 3 else 0
w = gen.get(name)
X = torch.from_numpy(gen.generate(w)).cuda()
for _ in range(reps):
    c = bm.cover_build(X, w.metric, w.eps, tile=tile)
    print(name, "L", c.L, "M", c.M, "E", c.E, "launches", c.stats.n_launches, flush=True)
    c.free()
torch.cuda.synchronize()
