#!/bin/bash
mkdir -p gpurun_out
L=abtmp/lib_wtrace.so
BM_LIB_PATH=$L BM_TC_TRACE=2 timeout 600 python tools/one_cover_path.py c5_l1 tensor 1 > gpurun_out/bo_wtrace.log 2>&1
grep wtrace gpurun_out/bo_wtrace.log | awk 'NR%60==30' | head -4
BM_LIB_PATH=$L BM_TC_TRACE=3 timeout 600 python tools/one_cover_path.py c5_l1 tensor 1 > gpurun_out/bo_tline.log 2>&1
grep tline gpurun_out/bo_tline.log | awk 'NR%60==30' | head -4
