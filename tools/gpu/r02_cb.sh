#!/bin/bash
# L1T epilogue with one tile of look-ahead: L1 parity tests, then same-box A/B against HEAD (lib_base)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "l1 or L1 or fullsize or validity" > gpurun_out/cb_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/cb_pytest.log
bash tools/ab_libs.sh "base la1" "c5_l1" 3
