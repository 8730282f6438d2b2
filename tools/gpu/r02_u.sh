#!/bin/bash
mkdir -p gpurun_out
for l in ${LIBS:-l128 l256}; do
  BM_LIB_PATH=abtmp/lib_${l}_w.so BM_TC_TRACE=3 timeout 300 python tools/one_cover.py ${W:-c5_cos} 1 > gpurun_out/u_tl_${l}.log 2>&1
  echo "== $l"; grep tline gpurun_out/u_tl_${l}.log | awk 'NR%20==3' | head -6
done
tools/ab_libs.sh "base l128 l256" "c5_cos c2" 3
