import json, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2601_01405_b200 as bm
from tests.helpers import case_arrays
cases = json.load(open("tests/golden/hand_examples.json"))["cases"]
only = sys.argv[1] if len(sys.argv) > 1 else None
for c in cases:
    if only and c["name"] != only: continue
    X, eps = case_arrays(c)
    print("case", c["name"], X.shape, X.dtype, c["metric"], flush=True)
    cov = bm.cover_build(torch.from_numpy(X).cuda(), c["metric"], eps)
    a = cov.numpy(); print("  ok", a["landmarks"].tolist(), flush=True)
