python tools/tc_probe.py > gpurun_out/tc_probe.txt 2>&1; cat gpurun_out/tc_probe.txt
