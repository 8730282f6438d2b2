"""One k_tc probe configuration (for ncu): python tools/tc_probe1.py n L mode"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_01405_b200 import bm as B  # noqa: E402

n, L, mode = (int(a) for a in sys.argv[1:4])
torch.manual_seed(0)
X = (torch.randn(n, 64) * 4).cuda()
print(B.tc_probe(X, L, mode, iters=2))
