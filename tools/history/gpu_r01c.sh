set -x
./tools/ubench/alu > gpurun_out/ubench_alu.txt 2>&1; cat gpurun_out/ubench_alu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
for w in c2 c1 c4; do timeout 600 python bench.py --workload $w --steps 10 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "bench $w rc=$?"; cat gpurun_out/bench_$w.json; tail -3 gpurun_out/bench_$w.err; done
timeout 600 python bench.py --workload c3_e8 --steps 3 --no-cpu-baseline > gpurun_out/bench_c3_e8.json 2> gpurun_out/bench_c3_e8.err; echo "bench c3 rc=$?"; cat gpurun_out/bench_c3_e8.json; tail -3 gpurun_out/bench_c3_e8.err
