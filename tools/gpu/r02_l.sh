#!/bin/bash
# wait-cycle traces (C5 cos, C3 eps=8), launch lists (C3 eps=8, C5 cos, C5 L1), ALU ubench, ncu of one C5 cos contraction
mkdir -p gpurun_out
(cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu alu.cu && ./alu) > gpurun_out/l_alu.txt 2>&1
for w in c5_cos c3_e8; do
  BM_LIB_PATH=paper_2601_01405_b200/libbm_b200_dbm_tc_wtrace.so BM_TC_TRACE=2 timeout 300 python tools/one_cover.py $w 1 > gpurun_out/l_wtrace_$w.log 2>&1
  echo "== $w"; grep wtrace gpurun_out/l_wtrace_$w.log | awk 'NR%10==5' | head -4
done
for w in c3_e8 c5_cos; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_launches_$w.csv \
     python tools/one_cover.py $w 1 > gpurun_out/l_ncu_$w.log 2>&1
  python tools/launch_summary.py gpurun_out/l_launches_$w.csv > gpurun_out/l_launches_$w.txt 2>&1; head -24 gpurun_out/l_launches_$w.txt
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tc" --kernel-name-base demangled \
   --launch-skip 40 --launch-count 1 -o gpurun_out/l_ncu_c5cos_member -f python tools/one_cover.py c5_cos 1 > gpurun_out/l_ncu1.log 2>&1
python tools/ncu_summary.py gpurun_out/l_ncu_c5cos_member.ncu-rep > gpurun_out/l_ncu_c5cos_member.txt 2>&1; head -30 gpurun_out/l_ncu_c5cos_member.txt
cat gpurun_out/l_alu.txt
