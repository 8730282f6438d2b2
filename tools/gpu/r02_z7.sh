#!/bin/bash
# ncu --set full of the C3 eps=8 contraction launches (A2 adjacency + pruned membership, one greedy tile)
O=gpurun_out/z7; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tc" \
   --launch-skip 60 --launch-count 2 -o $O/ncu_c3e8_tc -f python tools/one_cover.py c3_e8 1 > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/ncu_c3e8_tc.ncu-rep > $O/ncu_c3e8_tc.txt 2>&1; grep -n "kernel:\|duration\|DRAM read\|DRAM write\|tensor pipe\|issue active" $O/ncu_c3e8_tc.txt | head -20
