#!/bin/bash
# L1T levels per coordinate: B = 23 (12 K steps), 19 (10), 17 (9)
for v in kb378 kb314 kb282; do
  BM_LIB_PATH=abtmp/lib_$v.so timeout 600 python -m pytest tests/test_gpu_tensor.py -k "l1" -x -q -p no:cacheprovider 2>&1 | tail -1
  BM_LIB_PATH=abtmp/lib_$v.so BM_LOOP_PROFILE=1 timeout 900 python tools/one_cover_path.py c5_l1 auto 2 2>&1 | grep "loop profile" | tail -1
done
