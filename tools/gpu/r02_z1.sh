#!/bin/bash
# Re-entry baseline at HEAD: GPU suite, smoke, every bench line.
mkdir -p gpurun_out/z1
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/z1/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/z1/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/z1/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z1/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/z1/bench_c5_l1.json 2> gpurun_out/z1/bench_c5_l1.err; echo "bench rc=$?"
for w in c5_cos c3_e8 c3_e2 c4 c2; do
  timeout 900 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/z1/bench_$w.json 2> gpurun_out/z1/bench_$w.err
done
for w in c5_l1 c5_cos c3_e8 c3_e2 c4 c2; do
  python -c "
import json; d=json.load(open('gpurun_out/z1/bench_$w.json'))
print('$w', round(d['ms_per_step'],3), d['breakdown_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['seconds'])" || tail -3 gpurun_out/z1/bench_$w.err
done
