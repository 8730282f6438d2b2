#!/bin/bash
# L1 tensor path as the AUTO default: GPU suite, default bench line, the CUDA-core C5 L1 line, smoke
mkdir -p gpurun_out
BM_VALIDITY_LOG=gpurun_out/bp_validity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/bp_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/bp_pytest.log; tail -3 gpurun_out/bp_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bp_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bp_bench_default.json 2> gpurun_out/bp_bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --path cuda_core --steps 5 --no-cpu-baseline > gpurun_out/bp_bench_c5_l1_cc.json 2> gpurun_out/bp_bench_c5_l1_cc.err
for f in bp_bench_default bp_bench_c5_l1_cc; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); r=d['roofline']
print('$f', round(d['ms_per_step'],2), d['breakdown_ms'], 'frac', r['frac'], r.get('kernel'), 'e2e', d['e2e']['seconds'], 'cpu', (d.get('cpu_baseline') or {}).get('value'))"; done
