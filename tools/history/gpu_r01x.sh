python tools/step_var2.py c3_e8 10 > gpurun_out/stepvar6.log 2>&1; cat gpurun_out/stepvar6.log
python tools/step_var2.py c2 10 > gpurun_out/stepvar7.log 2>&1; cat gpurun_out/stepvar7.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
