#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tc<.*\(bool\)1>" --kernel-name-base demangled \
   --launch-skip 30 --launch-count 1 -o gpurun_out/d_ncu_c3e8_member -f python tools/one_cover.py c3_e8 1 > gpurun_out/d_ncu1.log 2>&1
tail -3 gpurun_out/d_ncu1.log
python tools/ncu_summary.py gpurun_out/d_ncu_c3e8_member.ncu-rep > gpurun_out/d_ncu_c3e8_member.txt 2>&1; head -40 gpurun_out/d_ncu_c3e8_member.txt
