#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/v_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/v_pytest.log
tools/ab_libs.sh "base l256b" "${W:-c5_cos c2 c3_e8}" 3
