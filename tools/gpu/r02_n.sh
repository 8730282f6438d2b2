#!/bin/bash
# parity of the tensor / L1 paths, then bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tensor.py -x -q -p no:cacheprovider > gpurun_out/n_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/n_pytest.log
for w in ${WL:-c5_cos c2 c5_l1}; do
  timeout 900 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/n_bench_$w.json 2> gpurun_out/n_bench_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/n_bench_$w.json'))
print('$w', round(d['ms_per_step'],3), d['breakdown_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['seconds'])" || tail -3 gpurun_out/n_bench_$w.err
done
