import sys, statistics, torch
sys.path.insert(0, ".")
import paper_2601_01405_b200 as bm
from workloads import gen
n = 5000
for D in (500, 1000, 200):
    eps = gen.cube_eps(D)
    Xs = [torch.from_numpy(gen.cube_cloud(n, D, t)).cuda() for t in range(20)]
    bm.cover_build(Xs[0], "l2", eps).free()
    ts = []
    for t in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); c = bm.cover_build(Xs[t], "l2", eps); b.record(); torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b), 2)); st = c.stats; c.free()
    print(D, ts, st.n_greedy_tiles, st.n_launches, flush=True)
