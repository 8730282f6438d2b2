"""Per-step phase times (library CUDA events) of repeated covers: which phase
carries the step-to-step variance."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2601_01405_b200 as bm  # noqa: E402
from workloads import gen  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = gen.get(name)
X = torch.from_numpy(gen.generate(w)).cuda()
s = torch.cuda.current_stream()
for _ in range(3):
    bm.cover_build(X, w.metric, w.eps).free()
for i in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    c = bm.cover_build(X, w.metric, w.eps, timing=True)
    b.record(s)
    st = c.stats.step_ms
    c.free()
    torch.cuda.synchronize()
    print(f"step {a.elapsed_time(b):8.1f} | " + " ".join(f"{k}={v:.1f}" for k, v in st.items()),
          flush=True)
