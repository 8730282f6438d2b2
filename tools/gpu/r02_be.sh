#!/bin/bash
# L1T: ncu --set full of one C5 L1 membership launch; per-phase loop profile
mkdir -p gpurun_out

timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_tc$" \
   --launch-skip 30 --launch-count 1 -o gpurun_out/bk_ncu_c5l1_l1t -f python tools/one_cover.py c5_l1 1 > gpurun_out/bk_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/bk_ncu.log
python tools/ncu_summary.py gpurun_out/bk_ncu_c5l1_l1t.ncu-rep > gpurun_out/bk_ncu_c5l1_l1t.txt 2>&1; cat gpurun_out/bk_ncu_c5l1_l1t.txt
