python tools/trace_run.py c5_l1 2 > gpurun_out/trace_c5.log 2>&1; tail -22 gpurun_out/trace_c5.log
