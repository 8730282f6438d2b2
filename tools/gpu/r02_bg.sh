#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tensor.py -k "l1" -x -q -p no:cacheprovider > gpurun_out/bd_pytest_l1.log 2>&1
echo "pytest l1 rc=$?"; tail -3 gpurun_out/bd_pytest_l1.log
timeout 900 python bench.py --workload c5_l1 --steps 3 --no-cpu-baseline > gpurun_out/bd_bench_c5_l1.json 2> gpurun_out/bd_bench_c5_l1.err
echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bd_bench_c5_l1.json')); print(d['ms_per_step'], d['breakdown_ms'], d['greedy'])"
L=abtmp/lib_wtrace.so
BM_LIB_PATH=$L BM_TC_TRACE=2 timeout 600 python tools/one_cover.py c5_l1 1 > gpurun_out/bf_wtrace.log 2>&1
grep wtrace gpurun_out/bf_wtrace.log | awk 'NR%40==20' | head -6
BM_LIB_PATH=$L BM_TC_TRACE=3 timeout 600 python tools/one_cover.py c5_l1 1 > gpurun_out/bf_tline.log 2>&1
grep -i "tline\|timeline" gpurun_out/bf_tline.log | awk 'NR%40==20' | head -6
