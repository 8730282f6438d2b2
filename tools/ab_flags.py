"""A/B of bm_options.flags on one workload: median device time of cover_build
(CUDA events, L2 flushed before each step) and the result sizes.
  python tools/ab_flags.py c2 0 8      # workload, flags..., (reps via --reps)"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2601_01405_b200 as bm  # noqa: E402
from workloads import gen  # noqa: E402

name = sys.argv[1]
flag_sets = [int(f) for f in sys.argv[2:]] or [0]
w = gen.get(name)
X = torch.from_numpy(gen.generate(w)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for fl in flag_sets:
    ts = []
    for r in range(13):
        flush.fill_(r & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        c = bm.cover_build(X, w.metric, w.eps, flags=fl)
        b.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(b))
        st = c.stats
        res = (c.L, c.M, c.E)
        c.free()
    print(f"{name} flags={fl}: median {statistics.median(ts):.4f} ms min {min(ts):.4f}  L,M,E={res}",
          f"tiles run/skip {st.tc_tiles_run}/{st.tc_tiles_skipped} chunks {st.tc_chunks_run}/{st.tc_chunks_skipped}",
          flush=True)
