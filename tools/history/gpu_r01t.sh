BM_TRACE=2 python tools/step_var2.py c3_e8 12 > gpurun_out/stepvar3.log 2>&1; cat gpurun_out/stepvar3.log
