for w in c5_l1; do timeout 900 python bench.py --workload $w --steps 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "bench $w rc=$?"; tail -3 gpurun_out/bench_$w.err; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "l1" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
