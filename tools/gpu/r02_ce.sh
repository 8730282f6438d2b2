#!/bin/bash
# L1T thermometer prep from byte-prefix masks (no per-byte loop): L1 parity tests, same-box A/B vs HEAD
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "l1 or L1" > gpurun_out/ce_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ce_pytest.log
bash tools/ab_libs.sh "chunk prep" "c5_l1" 3
