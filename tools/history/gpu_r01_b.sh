#!/bin/bash
# Round-1 late refresh: all bench lines, the oracle arm, the C2 launch list and
# ncu --set full captures of the dominant kernels (after each command exits 0 without ncu).
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -q -m gpu > gpurun_out/b_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py > gpurun_out/b_bench_c2.json 2> gpurun_out/b_bench_c2.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/b_ref_c2.json 2> gpurun_out/b_ref_c2.err; echo "ref rc=$?"
for w in c1 c4 c3_e2 c3_e4 c3_e8 c5_l1 c5_cos; do
  timeout 900 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/b_bench_$w.json 2> gpurun_out/b_bench_$w.err; echo "bench $w rc=$?"
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/b_plain_c2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b_launches_c2.csv $CMD > gpurun_out/b_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_tcILi0ELi1ELi256ELi1ELi4ELi3ELi0ELb1E" -s 6 -c 1 -o gpurun_out/b_prof_c2_tc $CMD > gpurun_out/b_ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
CMD3="python bench.py --workload c3_e8 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD3 > gpurun_out/b_plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_tcILi0ELi1ELi256ELi2ELi4ELi2ELi0ELb0E" -s 200 -c 1 -o gpurun_out/b_prof_c3_tc $CMD3 > gpurun_out/b_ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
CMD5="python bench.py --workload c5_cos --n 2000000 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD5 > gpurun_out/b_plain_c5cos.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_tcILi0ELi1ELi256ELi1ELi4ELi3ELi0ELb1E" -s 40 -c 1 -o gpurun_out/b_prof_c5cos_tc $CMD5 > gpurun_out/b_ncu_c5cos.log 2>&1; echo "ncu c5cos rc=$?"
python tools/bench_next.py --reps 3 --only color,skeleton > gpurun_out/b_next.jsonl 2> gpurun_out/b_next.err; echo "next rc=$?"
