#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tensor.py -x -q -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/q_pytest.log
tools/ab_libs.sh "${LIBS:-base lean32}" "${W:-c5_cos c2}" 3
