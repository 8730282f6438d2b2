#!/bin/bash
for l in sort4 sort5; do for r in 16 8; do echo "== $l rounds $r: $(BM_RS_ROUNDS=$r BM_LIB_PATH=abtmp/lib_$l.so python tools/sort_bench.py 140000000 39 5)"; done; done
