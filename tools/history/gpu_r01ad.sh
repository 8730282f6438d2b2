python tools/step_var2.py c2 25 > gpurun_out/stepvar8.log 2>&1; cat gpurun_out/stepvar8.log
