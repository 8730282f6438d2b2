#!/bin/bash
# round 2, call B: big-tile correctness + C3 timing
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "big_tile" > gpurun_out/b_pytest_big.log 2>&1
echo "rc=$?" >> gpurun_out/b_pytest_big.log
tail -5 gpurun_out/b_pytest_big.log
for w in c3_e8 c3_e2; do
  timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/b_bench_$w.json 2> gpurun_out/b_bench_$w.err
  tail -2 gpurun_out/b_bench_$w.err
  BM_LOOP_PROFILE=1 BM_TRACE=1 timeout 300 python -c "
import torch, paper_2601_01405_b200 as bm
from workloads import gen
w=gen.get('$w'); X=torch.from_numpy(gen.generate(w)).cuda()
for i in range(2): bm.cover_build(X, w.metric, w.eps).free()
" > gpurun_out/b_prof_$w.log 2>&1
  tail -40 gpurun_out/b_prof_$w.log
done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/b_pytest_all.log 2>&1
echo "rc=$?" >> gpurun_out/b_pytest_all.log
tail -5 gpurun_out/b_pytest_all.log
python - <<'PY'
import json
for w in ("c3_e8","c3_e2"):
    try:
        d=json.load(open(f"gpurun_out/b_bench_{w}.json"))
        print(w, d["ms_per_step"], d["breakdown_ms"], d["roofline"]["frac"], d["roofline"].get("other"), d["config"]["L"], d["greedy"])
    except Exception as e: print(w, e)
PY
