#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "edges or big_tile or full" > gpurun_out/y_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/y_pytest.log
for l in rows rows2k; do for w in c5_l1 c5_cos; do BM_ROWS_TRACE=1 BM_LIB_PATH=abtmp/lib_$l.so python tools/one_cover.py $w 1 2>&1 | grep "rows:"; done; done
tools/ab_libs.sh "pre rows rows2k" "${W:-c3_e8 c5_cos c5_l1}" 3
