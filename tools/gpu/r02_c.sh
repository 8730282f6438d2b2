#!/bin/bash
# round 2, call C: where does the C3 pruned membership kernel's time go
set -x
mkdir -p gpurun_out
BM_TC_TRACE=1 timeout 300 python tools/one_cover.py c3_e8 1 > gpurun_out/c_trace_c3e8.log 2>&1
grep -A 16 "membership tile 3[0-1]\]" gpurun_out/c_trace_c3e8.log | head -40
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tc" --kernel-name-base demangled \
   --launch-skip 60 --launch-count 1 -o gpurun_out/c_ncu_c3e8_member -f python tools/one_cover.py c3_e8 1 > gpurun_out/c_ncu1.log 2>&1
tail -3 gpurun_out/c_ncu1.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_launches_c3e8.csv \
   python tools/one_cover.py c3_e8 1 > gpurun_out/c_ncu2.log 2>&1
tail -3 gpurun_out/c_ncu2.log
python tools/launch_summary.py gpurun_out/c_launches_c3e8.csv > gpurun_out/c_launches_c3e8.txt 2>&1; head -30 gpurun_out/c_launches_c3e8.txt
python tools/ncu_summary.py gpurun_out/c_ncu_c3e8_member.ncu-rep > gpurun_out/c_ncu_c3e8_member.txt 2>&1; head -60 gpurun_out/c_ncu_c3e8_member.txt
