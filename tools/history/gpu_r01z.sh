for a in "3 0" "16 1" "3 1"; do timeout 120 python tools/repro_cos.py $a 2>&1 | tail -1; done
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/repro_cos.py 3 1 > gpurun_out/memcheck.log 2>&1; tail -40 gpurun_out/memcheck.log
