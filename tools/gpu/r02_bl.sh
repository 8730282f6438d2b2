#!/bin/bash
# GPU suite with the L1 tensor path; C4 contraction ncu capture (k_tc only)
mkdir -p gpurun_out
BM_VALIDITY_LOG=gpurun_out/bl_validity.jsonl timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/bl_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/bl_pytest.log; tail -3 gpurun_out/bl_pytest.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_tc$" \
   --launch-skip 8 --launch-count 1 -o gpurun_out/bl_ncu_c4_member -f python tools/one_cover.py c4 3 > gpurun_out/bl_ncu1.log 2>&1
python tools/ncu_summary.py gpurun_out/bl_ncu_c4_member.ncu-rep > gpurun_out/bl_ncu_c4_member.txt 2>&1; head -22 gpurun_out/bl_ncu_c4_member.txt
