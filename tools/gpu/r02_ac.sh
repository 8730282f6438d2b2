#!/bin/bash
for l in sort3 sort4; do echo "== $l"; for b in 39 56; do BM_LIB_PATH=abtmp/lib_$l.so python tools/sort_bench.py 140000000 $b 5; done; done
BM_LIB_PATH=abtmp/lib_sort4.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "radix or scan or edges or full_c4" 2>&1 | tail -1
