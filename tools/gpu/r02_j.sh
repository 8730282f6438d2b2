#!/bin/bash
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --show-backtrace device python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "dimension_widths and 33" > gpurun_out/j_san.log 2>&1
grep -m 30 -A 12 "Invalid\|Error\|error" gpurun_out/j_san.log | head -60
