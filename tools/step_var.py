"""Per-step device time of repeated covers under different harness settings
(diagnosing step-to-step variance): timing events on/off, L2 flush on/off,
nvidia-smi sampling on/off."""
import subprocess
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2601_01405_b200 as bm  # noqa: E402
from workloads import gen  # noqa: E402

name = sys.argv[1]
w = gen.get(name)
X = torch.from_numpy(gen.generate(w)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for _ in range(3):
    bm.cover_build(X, w.metric, w.eps).free()
for timing in (False, True):
    for fl in (False, True):
        for smi in (False, True):
            proc = None
            if smi:
                proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv",
                                         "-lms", "100"], stdout=subprocess.DEVNULL)
                time.sleep(0.3)
            ts = []
            for i in range(6):
                if fl:
                    flush.fill_(i)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                c = bm.cover_build(X, w.metric, w.eps, timing=timing)
                b.record(s)
                c.free()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            if proc:
                proc.terminate()
                proc.wait()
            print(f"timing={timing} flush={fl} smi={smi}: " + " ".join(f"{t:.1f}" for t in ts),
                  flush=True)
