set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
for w in c2 c1 c4; do timeout 600 python bench.py --workload $w --steps 10 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "bench $w rc=$?"; tail -3 gpurun_out/bench_$w.err; done
timeout 600 python bench.py --workload c3_e8 --steps 3 --no-cpu-baseline > gpurun_out/bench_c3_e8.json 2> gpurun_out/bench_c3_e8.err; echo "bench c3 rc=$?"; tail -3 gpurun_out/bench_c3_e8.err
timeout 300 python bench.py --workload c3_e8 --n 100000 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_tcILi" -s 20 -c 1 -o gpurun_out/prof_c3_tc2 python bench.py --workload c3_e8 --n 100000 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_c3.log 2>&1; echo "ncu c3 rc=$?"
