#!/bin/bash
# A/B: wait-cycle traces and bench of two library builds on the same box
mkdir -p gpurun_out
for l in ${LIBS:-base lean16}; do
  BM_LIB_PATH=abtmp/lib_${l}_w.so BM_TC_TRACE=2 timeout 300 python tools/one_cover.py ${W:-c5_cos} 1 > gpurun_out/o_wtrace_$l.log 2>&1
  echo "== $l"; grep wtrace gpurun_out/o_wtrace_$l.log | awk 'NR%20==10' | head -3
done
tools/ab_libs.sh "${LIBS:-base lean16}" "${W:-c5_cos}" 3
