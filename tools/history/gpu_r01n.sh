for w in c2 c1; do timeout 600 python bench.py --workload $w --steps 10 --path tensor --no-cpu-baseline > gpurun_out/bench_${w}_tc.json 2> gpurun_out/bench_${w}_tc.err; echo "bench $w rc=$?"; tail -3 gpurun_out/bench_${w}_tc.err; done
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c2_full or c1_full" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
