import math, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2601_01405_b200 as bm
from paper_2601_01405_b200 import bm as B
for seed in range(3):
    rng = np.random.default_rng([seed, 77])
    d, k = 24, 12
    centres = rng.normal(size=(k, d)) * 20.0
    X = (centres[rng.integers(0, k, size=9000)] + rng.normal(size=(9000, d))).astype(np.float32)
    eps = 3.0
    X[1::97] = X[0::97][: len(X[1::97])] + np.float32(eps / math.sqrt(d))
    t = torch.from_numpy(X).cuda()
    for tile in (256, 1024):
        a = bm.cover_build(t, "l2", eps, path="tensor", flags=B.FLAG_FORCE_PRUNE, tile=tile)
        b = bm.cover_build(t, "l2", eps, path="tensor", flags=B.FLAG_NO_PRUNE, tile=tile)
        s = a.stats
        print(seed, tile, "pruned L M E", a.L, a.M, a.E, "unpruned", b.L, b.M, b.E,
              "tiles run/skip", s.tc_tiles_run, s.tc_tiles_skipped, "chunks", s.tc_chunks_run, s.tc_chunks_skipped, "band", s.n_band_pairs, "ties", s.n_near_ties,
              flush=True)
