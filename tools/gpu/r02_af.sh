#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/af_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/af_pytest.log
python tools/sort_bench.py 140000000 39 5
python tools/sort_bench.py 640000000 38 3
tools/ab_libs.sh "pre cur" "c3_e8 c5_cos c5_l1" 2
