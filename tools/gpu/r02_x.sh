#!/bin/bash
for r in 16 8 4; do BM_RS_ROUNDS=$r python tools/sort_bench.py 140000000 39 5; done
