#!/bin/bash
mkdir -p gpurun_out
echo "== a"; timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_tensor.py -q -p no:cacheprovider -k "(c5_l1 and tensor) or clusters" 2>&1 | tail -2
echo "== b"; timeout 900 python -m pytest tests/test_gpu_tensor.py -q -p no:cacheprovider -k "clusters" 2>&1 | tail -2
echo "== c"; timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_tensor.py -q -p no:cacheprovider -k "(c5_l1 and auto) or clusters" 2>&1 | tail -2
echo "== d"; timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_tensor.py -q -p no:cacheprovider -k "c3_e8 or clusters" 2>&1 | tail -2
