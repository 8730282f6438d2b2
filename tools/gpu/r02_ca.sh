#!/bin/bash
# re-entry baseline at HEAD (after the L1T 20-level and radix-hist commits): GPU suite, smoke, bench lines
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ca_smi.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/ca_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ca_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ca_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/ca_bench_c5_l1.json 2> gpurun_out/ca_bench_c5_l1.err; echo "default rc=$?"
for w in c5_cos c3_e8 c3_e2 c4 c2; do
  timeout 900 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/ca_bench_$w.json 2> gpurun_out/ca_bench_$w.err; echo "$w rc=$?"
done
for f in gpurun_out/ca_bench_*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']
print('$f'.split('ca_bench_')[1], round(d['ms_per_step'],3), d.get('breakdown_ms'), 'frac', r['frac'], 'e2e', d['e2e']['seconds'])"; done
