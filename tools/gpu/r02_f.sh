#!/bin/bash
mkdir -p gpurun_out
for w in c3_e2 c3_e8 c5_cos c2; do
  BM_TC_TRACE=2 timeout 300 python tools/one_cover.py $w 1 > gpurun_out/f_wtrace_$w.log 2>&1
  echo "== $w"; grep wtrace gpurun_out/f_wtrace_$w.log | awk 'NR%20==5' | head -4
done
