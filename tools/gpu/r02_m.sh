#!/bin/bash
# ncu --set full with source of one C5 cos contraction and one C5 L1 membership launch
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tc<" --kernel-name-base demangled \
   --launch-skip 60 --launch-count 1 -o gpurun_out/m_ncu_c5cos_member -f python tools/one_cover.py c5_cos 1 > gpurun_out/m_ncu1.log 2>&1
python tools/ncu_summary.py gpurun_out/m_ncu_c5cos_member.ncu-rep > gpurun_out/m_ncu_c5cos_member.txt 2>&1; head -24 gpurun_out/m_ncu_c5cos_member.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_pairs<1" --kernel-name-base demangled \
   --launch-skip 150 --launch-count 1 -o gpurun_out/m_ncu_c5l1_member -f python tools/one_cover.py c5_l1 1 > gpurun_out/m_ncu2.log 2>&1
python tools/ncu_summary.py gpurun_out/m_ncu_c5l1_member.ncu-rep > gpurun_out/m_ncu_c5l1_member.txt 2>&1; head -24 gpurun_out/m_ncu_c5l1_member.txt
tail -3 gpurun_out/m_ncu1.log gpurun_out/m_ncu2.log
