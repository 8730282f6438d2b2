#!/bin/bash
mkdir -p gpurun_out
for i in 1 2 3; do
timeout 600 python -m pytest tests/test_gpu_tensor.py -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_tensor.py -q -p no:cacheprovider -k "l1 or pruned" 2>&1 | tail -2
done
