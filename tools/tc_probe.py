"""Where does the tcgen05 contraction's time go?  Times k_tc (tf32, d=64) with
the full membership epilogue (mode 0), an epilogue that only reads TMEM
(mode 2) and one that releases TMEM unread (mode 3)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_01405_b200 import bm as B  # noqa: E402

torch.manual_seed(0)
for n, L in ((1_000_000, 1024), (200_000, 16384)):
    X = (torch.randn(n, 64) * 4).cuda()
    for cfg in (0, 1):
        for mode in (0, 2, 3):
            ms = B.tc_probe(X, L, mode + 16 * cfg, iters=5)
            tf = 2.0 * 64 * n * L / (ms * 1e-3) / 1e12
            print(f"n={n} L={L} cfg={cfg} mode={mode}: {ms:.3f} ms  {tf:.1f} TFLOP/s (tf32 ~832)")
