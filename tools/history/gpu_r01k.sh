timeout 300 python bench.py --workload c3_e8 --n 200000 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c3p.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3p.csv python bench.py --workload c3_e8 --n 200000 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c3p.log 2>&1; echo "ncu rc=$?"
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
