#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tensor.py tests/test_gpu_fullsize.py -k "l1" -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bt_bench.json 2> gpurun_out/bt_bench.err; python -c "
import json; d=json.load(open('gpurun_out/bt_bench.json')); r=d['roofline']
print(round(d['ms_per_step'],2), d['breakdown_ms'], 'frac', r['frac'], r['peak'], 'e2e', d['e2e']['seconds'])"
