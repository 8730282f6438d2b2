#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tensor.py tests/test_gpu_next.py -x -q -p no:cacheprovider > gpurun_out/i_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/i_pytest.log
tools/ab_libs.sh "${LIBS:-live cur}" "${WL:-c3_e8 c3_e2 c5_cos c2}" 5
