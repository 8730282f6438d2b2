"""Run a few covers of a workload with BM_TRACE=1 (per-sub-step host timings)."""
import os
import sys

os.environ["BM_TRACE"] = "1"
sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2601_01405_b200 as bm  # noqa: E402
from workloads import gen  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = gen.get(name)
X = torch.from_numpy(gen.generate(w)).cuda()
for r in range(reps):
    print(f"--- {name} run {r}", file=sys.stderr, flush=True)
    c = bm.cover_build(X, w.metric, w.eps)
    print(f"L={c.L} M={c.M} E={c.E} P={c.P}", file=sys.stderr, flush=True)
    c.free()
