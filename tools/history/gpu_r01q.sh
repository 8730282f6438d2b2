python tools/trace_run.py c3_e8 4 > gpurun_out/trace_c3.log 2>&1; tail -60 gpurun_out/trace_c3.log
