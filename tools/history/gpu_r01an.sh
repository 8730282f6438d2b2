CMD="python bench.py --workload c5_l1 --n 2000000 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_c5p.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_rs_scatterILi16E" -s 20 -c 1 -o gpurun_out/prof_rs $CMD > gpurun_out/ncu_rs.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_rs.log
