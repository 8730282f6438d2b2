#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tensor.py -k "l1" -x -q -p no:cacheprovider > gpurun_out/bd_pytest_l1.log 2>&1
echo "pytest l1 rc=$?"; tail -3 gpurun_out/bd_pytest_l1.log
timeout 900 python bench.py --workload c5_l1 --steps 3 --no-cpu-baseline > gpurun_out/bd_bench_c5_l1.json 2> gpurun_out/bd_bench_c5_l1.err
echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bd_bench_c5_l1.json')); print(d['ms_per_step'], d['breakdown_ms'], d['greedy'])"
