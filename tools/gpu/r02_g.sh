#!/bin/bash
mkdir -p gpurun_out
for w in c3_e2 c5_cos; do
  BM_TC_TRACE=2 timeout 300 python tools/one_cover.py $w 1 > gpurun_out/g_wtrace_$w.log 2>&1
  echo "== $w"; grep wtrace gpurun_out/g_wtrace_$w.log | awk 'NR%20==5' | head -3
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tc<.*\(bool\)1>" --kernel-name-base demangled \
   --launch-skip 40 --launch-count 1 -o gpurun_out/g_ncu_c3e2_member -f python tools/one_cover.py c3_e2 1 > gpurun_out/g_ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tc<.*\(bool\)1, \(bool\)0>" --kernel-name-base demangled \
   --launch-skip 40 --launch-count 1 -o gpurun_out/g_ncu_c5cos_member -f python tools/one_cover.py c5_cos 1 > gpurun_out/g_ncu2.log 2>&1
tail -2 gpurun_out/g_ncu1.log gpurun_out/g_ncu2.log
