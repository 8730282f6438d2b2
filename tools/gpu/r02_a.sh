#!/bin/bash
# round 2, call A: GPU test suite (incl. full-size validity), tcgen05 peaks, default bench
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt
(cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_peak tc_peak.cu && ./tc_peak) > gpurun_out/tc_peak.json 2>&1
BM_VALIDITY_LOG=gpurun_out/validity.jsonl timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=25 > gpurun_out/a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/a_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/a_bench_c5_l1.json 2> gpurun_out/a_bench_c5_l1.err
tail -3 gpurun_out/a_pytest.log
cat gpurun_out/tc_peak.json gpurun_out/a_bench_c5_l1.json
