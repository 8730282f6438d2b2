#!/bin/bash
# Round-1 late refresh (after tile-level pruning): all bench lines, the oracle
# arm, launch list and ncu --set full of the pruned C3 contraction.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -q -m gpu > gpurun_out/c_pytest_gpu.log 2>&1; echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/c_bench_c2.json 2> gpurun_out/c_bench_c2.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/c_ref_c2.json 2> gpurun_out/c_ref_c2.err; echo "ref rc=$?"
for w in c1 c4 c3_e2 c3_e4 c3_e8 c5_l1 c5_cos; do
  timeout 900 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/c_bench_$w.json 2> gpurun_out/c_bench_$w.err; echo "bench $w rc=$?"
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/c_plain_c2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_launches_c2.csv $CMD > gpurun_out/c_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
CMD3="python bench.py --workload c3_e8 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD3 > gpurun_out/c_plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_tcILi0ELi1ELi256ELi2ELi3ELi3ELi0ELb0E" -s 200 -c 1 -o gpurun_out/c_prof_c3_tc $CMD3 > gpurun_out/c_ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
