timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "radix or c2_full or prefix" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
python tools/trace_run.py c5_l1 2 > gpurun_out/trace_c5.log 2>&1; grep -E "sort|emit|compact" gpurun_out/trace_c5.log | tail -5
