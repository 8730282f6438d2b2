python tools/tc_probe1.py 1000000 1024 0 > gpurun_out/p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_tcILi0ELi1ELi256ELi2ELi4ELi2ELi0E" -s 1 -c 1 -o gpurun_out/prof_probe0 python tools/tc_probe1.py 1000000 1024 0 > gpurun_out/ncu_probe.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_probe.log
