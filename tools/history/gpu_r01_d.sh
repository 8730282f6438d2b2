#!/bin/bash
# Round-1 final refresh: GPU tests, smoke, every bench line, the oracle arm,
# the §8(f) rows, the paper grid, the C2 launch list and an ncu --set full
# capture of the C2 membership kernel.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/d_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/d_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/d_bench_c2.json 2> gpurun_out/d_bench_c2.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/d_ref_c2.json 2> gpurun_out/d_ref_c2.err; echo "ref rc=$?"
for w in c1 c4 c3_e2 c3_e4 c3_e8 c5_l1 c5_cos; do
  timeout 900 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/d_bench_$w.json 2> gpurun_out/d_bench_$w.err; echo "bench $w rc=$?"
done
timeout 900 python tools/paper_grid.py --trials 65 --oracle-trials 3 --out gpurun_out/d_paper_grid.jsonl > gpurun_out/d_paper_grid.log 2>&1; echo "grid rc=$?"
timeout 1200 python tools/bench_next.py --reps 5 > gpurun_out/d_next.jsonl 2> gpurun_out/d_next.err; echo "next rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/d_plain_c2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d_launches_c2.csv $CMD > gpurun_out/d_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k k_tc -s 10 -c 1 -o gpurun_out/d_prof_c2_tc $CMD > gpurun_out/d_ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
