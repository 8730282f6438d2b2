#!/bin/bash
# L1T epilogue groups A/B (4 groups x 64 columns vs 2 groups x 128 columns), same box
mkdir -p gpurun_out
for v in base cl; do
  BM_LIB_PATH=abtmp/lib_$v.so timeout 600 python -m pytest tests/test_gpu_tensor.py -k "l1" -x -q -p no:cacheprovider 2>&1 | tail -1
  BM_LIB_PATH=abtmp/lib_$v.so BM_LOOP_PROFILE=1 timeout 900 python tools/one_cover_path.py c5_l1 tensor 2 2>&1 | tail -2
done
