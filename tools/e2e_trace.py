"""Host-buffer (e2e) covers of one workload with per-call wall time; run with
BM_TRACE=3 for the library's host timestamps.  python tools/e2e_trace.py c2 [reps]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2601_01405_b200 as bm  # noqa: E402
from workloads import gen  # noqa: E402

w = gen.get(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
X = torch.from_numpy(gen.generate(w)).pin_memory()
for r in range(reps):
    print(f"--- run {r}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    c = bm.cover_build_host(X, w.metric, w.eps)
    print(f"e2e {1e3 * (time.perf_counter() - t0):.3f} ms L={c.L}", file=sys.stderr, flush=True)
    c.free()
