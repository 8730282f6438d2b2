python tools/step_var2.py c3_e8 12 > gpurun_out/stepvar2.log 2>&1; cat gpurun_out/stepvar2.log
