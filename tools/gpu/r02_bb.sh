#!/bin/bash
# L1 on tensor cores: new parity tests, the C5 L1 bench line, full-size validity of C5 L1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tensor.py -k "l1" -x -q -p no:cacheprovider > gpurun_out/bb_pytest_l1.log 2>&1
echo "pytest l1 rc=$?"; tail -15 gpurun_out/bb_pytest_l1.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -k "near_tie" -x -q -p no:cacheprovider > gpurun_out/bb_pytest_tie.log 2>&1
echo "pytest tie rc=$?"; tail -3 gpurun_out/bb_pytest_tie.log
timeout 900 python bench.py --workload c5_l1 --steps 3 --no-cpu-baseline > gpurun_out/bb_bench_c5_l1.json 2> gpurun_out/bb_bench_c5_l1.err
echo "bench rc=$?"; tail -c 1500 gpurun_out/bb_bench_c5_l1.json; tail -5 gpurun_out/bb_bench_c5_l1.err
BM_VALIDITY_LOG=gpurun_out/bb_validity.jsonl timeout 1500 python -m pytest tests/test_gpu_fullsize.py -k "c5_l1" -x -q -p no:cacheprovider > gpurun_out/bb_pytest_full.log 2>&1
echo "pytest full rc=$?"; tail -3 gpurun_out/bb_pytest_full.log
