#!/bin/bash
cat > /tmp/chain.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2601_01405_b200 as bm
X = torch.from_numpy(np.arange(20000, dtype=np.float32).reshape(-1, 1)).cuda()
rng = np.random.default_rng(9)
Y = (rng.random((12000, 3)) * 0.2).astype(np.float32); Y[6000:] += 5.0 * rng.random((6000, 3)).astype(np.float32)
Y = torch.from_numpy(Y).cuda()
bad = 0
for r in range(int(sys.argv[1])):
    try:
        a = bm.cover_build(X, "l2", 1.5, tile=8192, path="tensor"); a.free()
        b = bm.cover_build(Y, "l2", 0.05, tile=8192, path="tensor"); b.free()
    except Exception as e:
        print("ERR", r, str(e)[:150]); bad += 1; break
print("done", bad)
PY
for l in rows; do echo "== $l"; BM_LIB_PATH=abtmp/lib_$l.so timeout 600 python /tmp/chain.py 200 2>&1 | tail -2; done
