#!/bin/bash
# flaky pruned-cluster test: old (f6fe16b) vs new library, 12 runs each
for v in old new; do
  f=0
  for i in $(seq 1 12); do
    BM_LIB_PATH=abtmp/lib_$v.so timeout 300 python -m pytest tests/test_gpu_tensor.py -q -p no:cacheprovider -k "clusters" > /tmp/r.log 2>&1 || { f=$((f+1)); grep FAILED /tmp/r.log | head -2; }
  done
  echo "$v failures: $f / 12"
done
