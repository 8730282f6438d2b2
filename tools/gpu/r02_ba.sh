#!/bin/bash
# re-entry (session 3): GPU suite, smoke, the default bench line (with the oracle baseline),
# C4 / C3 eps=8 lines, C3 eps=8 + C5 L1 launch lists, ncu --set full of one C4 contraction
# and of the HBM passes (sort / unique / prep / row pairs) on C5 L1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ba_smi.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/ba_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ba_pytest.log; tail -2 gpurun_out/ba_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ba_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/ba_bench_default.json 2> gpurun_out/ba_bench_default.err; echo "bench rc=$?"
for w in c4 c3_e8; do
  timeout 900 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/ba_bench_$w.json 2> gpurun_out/ba_bench_$w.err
done
for w in c3_e8 c5_l1; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ba_launches_$w.csv \
     python tools/one_cover.py $w 1 > gpurun_out/ba_ncu_l_$w.log 2>&1
  python tools/launch_summary.py gpurun_out/ba_launches_$w.csv > gpurun_out/ba_launches_$w.txt 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tc" \
   --launch-skip 20 --launch-count 1 -o gpurun_out/ba_ncu_c4_member -f python tools/one_cover.py c4 3 > gpurun_out/ba_ncu1.log 2>&1
python tools/ncu_summary.py gpurun_out/ba_ncu_c4_member.ncu-rep > gpurun_out/ba_ncu_c4_member.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_rs_|k_unique|k_row_pairs|k_prep|k_segment|k_unpack|k_l1_quant" \
   --launch-count 14 -o gpurun_out/ba_ncu_c5l1_hbm -f python tools/one_cover.py c5_l1 1 > gpurun_out/ba_ncu2.log 2>&1
python tools/ncu_summary.py gpurun_out/ba_ncu_c5l1_hbm.ncu-rep > gpurun_out/ba_ncu_c5l1_hbm.txt 2>&1
ls gpurun_out
