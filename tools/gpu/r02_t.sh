#!/bin/bash
mkdir -p gpurun_out
for l in ${LIBS:-dA dB dC}; do
  BM_LIB_PATH=abtmp/lib_${l}_w.so BM_TC_TRACE=3 timeout 300 python tools/one_cover.py ${W:-c5_cos} 1 > gpurun_out/t_tl_${l}.log 2>&1
  echo "== $l"; grep tline gpurun_out/t_tl_${l}.log | awk 'NR%10==3' | head -4; tail -1 gpurun_out/t_tl_${l}.log
done
