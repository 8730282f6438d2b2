"""C2-shaped probe of the tcgen05 contraction (n = 1e5, d = 10, the C2 torus
rows): full membership epilogue (mode 0), TMEM reads only (2), TMEM released
unread (3), for landmark tiles of 256 / 512 / 768 columns; then one traced
launch per L (per-CTA %globaltimer stamps of the kernel's phases, stderr)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_01405_b200 import bm as B  # noqa: E402
from workloads import gen  # noqa: E402

X = torch.from_numpy(gen.generate(gen.get("c2"))).cuda()
for L in (256, 512, 768, 1024):
    for mode in (0, 2, 3, 32, 34, 35):   # + 32: resident-B instance
        ms = B.tc_probe(X, L, mode, iters=20)
        print(f"c2 n={X.shape[0]} L={L} mode={mode}: {ms * 1e3:.1f} us", flush=True)
    B.tc_probe(X, L, 256 + 32, iters=5)
    sys.stderr.flush()
