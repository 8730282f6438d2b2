set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/fin_bench_c2.json 2> gpurun_out/fin_bench_c2.err; echo "rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/fin_ref_c2.json 2> gpurun_out/fin_ref_c2.err; echo "rc=$?"
for w in c1 c4 c3_e2 c3_e4 c3_e8 c5_l1 c5_cos; do timeout 900 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/fin_bench_$w.json 2> gpurun_out/fin_bench_$w.err; echo "bench $w rc=$?"; done
