#!/bin/bash
# Final check of the closing tree: GPU suite, smoke, default bench line, C3 eps=8 line, then the C3 contraction capture
O=gpurun_out/z8; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_c5_l1.json 2> $O/bench_c5_l1.err; echo "bench rc=$?"
timeout 900 python bench.py --workload c3_e8 > $O/bench_c3_e8.json 2> $O/bench_c3_e8.err
for w in c5_l1 c3_e8; do
  python -c "
import json; d=json.load(open('$O/bench_$w.json'))
print('$w', round(d['ms_per_step'],3), d['breakdown_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['seconds'])" || tail -3 $O/bench_$w.err
done
bash tools/gpu/r02_z7.sh
