#!/bin/bash
mkdir -p gpurun_out
python tools/sort_bench.py 140000000 39 5
python tools/sort_bench.py 640000000 38 3
python tools/sort_bench.py 98000000 56 3
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rs_scatter" --launch-skip 7 --launch-count 1 -o gpurun_out/w_ncu_rs_scatter -f python tools/sort_bench.py 140000000 39 1 > gpurun_out/w_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rs_hist" --launch-skip 1 --launch-count 1 -o gpurun_out/w_ncu_rs_hist -f python tools/sort_bench.py 140000000 39 1 > gpurun_out/w_ncu2.log 2>&1
python tools/ncu_summary.py gpurun_out/w_ncu_rs_scatter.ncu-rep | head -20
python tools/ncu_summary.py gpurun_out/w_ncu_rs_hist.ncu-rep | head -8
