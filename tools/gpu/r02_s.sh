#!/bin/bash
mkdir -p gpurun_out
BM_LIB_PATH=abtmp/lib_bn128.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tensor.py -x -q -p no:cacheprovider > gpurun_out/s_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s_pytest.log
for l in ${LIBS:-bn128}; do
  for w in ${W:-c5_cos}; do
  BM_LIB_PATH=abtmp/lib_${l}_w.so BM_TC_TRACE=3 timeout 300 python tools/one_cover.py $w 1 > gpurun_out/s_tl_${l}_$w.log 2>&1
  echo "== $l $w"; grep tline gpurun_out/s_tl_${l}_$w.log | awk 'NR%10==3' | head -4
  done
done
tools/ab_libs.sh "base bn128" "c5_cos c2" 3
