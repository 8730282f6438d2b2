#!/bin/bash
# C4: one column chunk per row block for the single-A-buffer instance (A/B vs HEAD); the C4 parity
# tests; launch list of the default bench command; ncu --set full (with L2 / stall metrics) of one
# C5 L1 and one C4 contraction launch
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "c4 or C4 or int or u8 or i8" > gpurun_out/cd_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/cd_pytest.log
bash tools/ab_libs.sh "base chunk" "c4" 10
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cd_launches_default.csv $CMD > gpurun_out/cd_ncu_launch.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/cd_launches_default.csv > gpurun_out/cd_launches_default.txt 2>&1; head -8 gpurun_out/cd_launches_default.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_tc$" \
   --launch-skip 60 --launch-count 1 -o gpurun_out/cd_ncu_c5l1_member -f python tools/one_cover.py c5_l1 1 > gpurun_out/cd_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/cd_ncu_c5l1_member.ncu-rep > gpurun_out/cd_ncu_c5l1_member.txt 2>&1; head -30 gpurun_out/cd_ncu_c5l1_member.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_tc$" \
   --launch-skip 9 --launch-count 1 -o gpurun_out/cd_ncu_c4_member -f python tools/one_cover.py c4 2 > gpurun_out/cd_ncu4.log 2>&1
python tools/ncu_summary.py gpurun_out/cd_ncu_c4_member.ncu-rep > gpurun_out/cd_ncu_c4_member.txt 2>&1; head -30 gpurun_out/cd_ncu_c4_member.txt
