#!/bin/bash
# quick loop: tensor / big-tile tests, C3 benches, C3 e8 launch list
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tensor.py -x -q -p no:cacheprovider > gpurun_out/e_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/e_pytest.log
tail -3 gpurun_out/e_pytest.log
for w in ${WL:-c3_e8 c3_e2}; do
  timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/e_bench_$w.json 2> gpurun_out/e_bench_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/e_bench_$w.json'))
print('$w', round(d['ms_per_step'],3), d['breakdown_ms'], 'frac', d['roofline']['frac'], d['roofline']['other']['executed_tiles'] if 'other' in d['roofline'] else '', 'e2e', d['e2e']['seconds'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e_launches_c3e8.csv \
   python tools/one_cover.py c3_e8 1 > gpurun_out/e_ncu2.log 2>&1
python tools/launch_summary.py gpurun_out/e_launches_c3e8.csv > gpurun_out/e_launches_c3e8.txt 2>&1; head -16 gpurun_out/e_launches_c3e8.txt
