#!/bin/bash
BM_LIB_PATH=abtmp/lib_sort3.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rs_scatter" --launch-skip 7 --launch-count 1 -o gpurun_out/ad_ncu_rs -f python tools/sort_bench.py 140000000 39 1 > gpurun_out/ad_ncu.log 2>&1
tail -1 gpurun_out/ad_ncu.log
