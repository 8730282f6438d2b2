CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_c2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_tcILi0ELi1ELi256ELi2ELi4ELi2ELi0E" -s 6 -c 1 -o gpurun_out/fin_prof_c2_tc $CMD > gpurun_out/ncu_full_c2.log 2>&1; echo "ncu2 rc=$?"
CMD3="python bench.py --workload c3_e8 --n 100000 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD3 > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_tcILi0ELi1ELi256ELi2ELi4ELi2ELi0E" -s 30 -c 1 -o gpurun_out/fin_prof_c3_tc $CMD3 > gpurun_out/ncu_full_c3.log 2>&1; echo "ncu3 rc=$?"
