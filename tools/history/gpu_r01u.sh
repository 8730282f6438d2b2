BM_POOL=0 python tools/step_var2.py c3_e8 12 > gpurun_out/stepvar4.log 2>&1; cat gpurun_out/stepvar4.log
nvidia-smi -q | grep -i -A3 "compute mode\|persistence\|MIG" | head -20
ps aux | grep -v grep | grep -i -E "nvidia|python" | head
