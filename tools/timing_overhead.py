"""Step time with and without the library's per-step timing events (which sit
between kernels of the tile loop)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2601_01405_b200 as bm  # noqa: E402
from workloads import gen  # noqa: E402

for name in sys.argv[1:] or ["c2"]:
    w = gen.get(name)
    X = torch.from_numpy(gen.generate(w)).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for timing in (True, False, True, False):
        for _ in range(3):
            bm.cover_build(X, w.metric, w.eps, timing=timing).free()
        ts = []
        for i in range(20):
            flush.fill_(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            c = bm.cover_build(X, w.metric, w.eps, timing=timing)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
            c.free()
        ts.sort()
        print(name, "timing" if timing else "plain ", "median %.4f ms  min %.4f" % (ts[10], ts[0]))
