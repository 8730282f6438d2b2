#!/bin/bash
# ncu source-level capture of one C5-cosine contraction launch (2e6 prefix)
CMD="python bench.py --workload c5_cos --n 2000000 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_c5cos.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_tcILi0ELi1ELi256ELi1ELi4ELi3ELi0ELb1E" -s 40 -c 1 -o gpurun_out/aw_c5cos_tc $CMD > gpurun_out/ncu_au.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_au.log
