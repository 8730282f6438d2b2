"""One paper-grid cell, diagnostics: path, tiles, band pairs, device time.
  python tools/grid_cell.py N D [D ...]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2601_01405_b200 as bm  # noqa: E402
from workloads import gen  # noqa: E402

n = int(sys.argv[1])
for D in map(int, sys.argv[2:]):
    eps = gen.cube_eps(D)
    X = torch.from_numpy(gen.cube_cloud(n, D, 0)).cuda()
    ts = []
    for r in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        c = bm.cover_build(X, "l2", eps, timing=(r == 7))
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        st = c.stats
        c.free()
    print(f"n={n} D={D} eps={eps:.3f} path={st.path_used} L={st.L if hasattr(st,'L') else ''} "
          f"band={st.n_band_pairs} ties={st.n_near_ties} tiles={st.n_greedy_tiles} launches={st.n_launches} ms med={statistics.median(ts[:7]):.3f} all={[round(t, 2) for t in ts]} "
          f"steps={ {k: round(v, 3) for k, v in st.step_ms.items()} }", flush=True)
