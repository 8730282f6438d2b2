python tools/step_var.py c3_e8 > gpurun_out/stepvar.log 2>&1; cat gpurun_out/stepvar.log
