#!/bin/bash
mkdir -p gpurun_out
for l in ${LIBS:-base lean32}; do
  for w in ${W:-c5_cos c2}; do
  BM_LIB_PATH=abtmp/lib_${l}_w.so BM_TC_TRACE=3 timeout 300 python tools/one_cover.py $w 1 > gpurun_out/r_tl_${l}_$w.log 2>&1
  echo "== $l $w"; grep tline gpurun_out/r_tl_${l}_$w.log | awk 'NR%10==3' | head -4
  done
done
