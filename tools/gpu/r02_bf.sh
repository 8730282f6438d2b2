#!/bin/bash
# L1T diagnostics: per-role wait cycles and CTA 0's tile timeline (diagnostic build)
mkdir -p gpurun_out
L=abtmp/lib_wtrace.so
BM_LIB_PATH=$L BM_TC_TRACE=2 timeout 600 python tools/one_cover.py c5_l1 1 > gpurun_out/bf_wtrace.log 2>&1
grep wtrace gpurun_out/bf_wtrace.log | awk 'NR%40==20' | head -6
BM_LIB_PATH=$L BM_TC_TRACE=3 timeout 600 python tools/one_cover.py c5_l1 1 > gpurun_out/bf_tline.log 2>&1
grep -i "tline\|timeline" gpurun_out/bf_tline.log | awk 'NR%40==20' | head -6
