#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tensor.py -x -q -p no:cacheprovider > gpurun_out/h_pytest.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/h_pytest.log
for w in c3_e2 c3_e8 c5_cos; do
  BM_TC_TRACE=2 timeout 300 python tools/one_cover.py $w 1 > gpurun_out/h_wtrace_$w.log 2>&1
  echo "== $w"; grep wtrace gpurun_out/h_wtrace_$w.log | awk 'NR%20==5' | head -2
done
for w in ${WL:-c3_e8 c3_e2}; do
  timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/h_bench_$w.json 2> gpurun_out/h_bench_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/h_bench_$w.json'))
print('$w', round(d['ms_per_step'],3), d['breakdown_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['seconds'])"
done
