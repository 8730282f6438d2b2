"""Run N covers of a workload on a given path (diagnostics / A-B of library builds):
python tools/one_cover_path.py c5_l1 tensor [N]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_01405_b200 as bm  # noqa: E402
from workloads import gen  # noqa: E402

name, path = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = gen.get(name)
X = torch.from_numpy(gen.generate(w)).cuda()
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c = bm.cover_build(X, w.metric, w.eps, path=path)
    t1 = time.perf_counter()
    print(name, path, "L", c.L, "M", c.M, "E", c.E, "wall_ms %.1f" % ((t1 - t0) * 1e3), flush=True)
    c.free()
