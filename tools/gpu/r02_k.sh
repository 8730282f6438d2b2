#!/bin/bash
# re-entry baseline at HEAD: GPU suite, smoke, every workload's bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/k_smi.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/k_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/k_pytest.log; tail -3 gpurun_out/k_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/k_smoke.log 2>&1; echo "smoke rc=$?"
for w in c5_l1 c3_e8 c3_e2 c5_cos c4 c2; do
  timeout 900 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/k_bench_$w.json 2> gpurun_out/k_bench_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/k_bench_$w.json'))
print('$w', round(d['ms_per_step'],3), d['breakdown_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['seconds'])" || tail -3 gpurun_out/k_bench_$w.err
done
