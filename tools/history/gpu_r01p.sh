for w in c5_l1 c3_e8; do timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "bench $w rc=$?"; tail -3 gpurun_out/bench_$w.err; done
timeout 300 python bench.py --workload c5_l1 --n 2000000 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5p.csv python bench.py --workload c5_l1 --n 2000000 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c5p.log 2>&1; echo "ncu rc=$?"
