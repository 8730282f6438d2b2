python tools/tc_probe.py > gpurun_out/tc_probe.txt 2>&1; head -3 gpurun_out/tc_probe.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for w in c3_e8 c2; do timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "bench $w rc=$?"; tail -3 gpurun_out/bench_$w.err; done
