#!/bin/bash
mkdir -p gpurun_out
BM_LIB_PATH=abtmp/lib_${L:-lean16}.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tc<" --kernel-name-base demangled \
   --launch-skip 60 --launch-count 1 -o gpurun_out/p_ncu_c5cos_${L:-lean16} -f python tools/one_cover.py c5_cos 1 > gpurun_out/p_ncu1.log 2>&1
python tools/ncu_summary.py gpurun_out/p_ncu_c5cos_${L:-lean16}.ncu-rep 2>&1 | head -20
