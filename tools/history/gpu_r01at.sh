#!/bin/bash
# warp-aggregated key emission in the contraction epilogue
timeout 600 python -m pytest tests/test_gpu_tensor.py tests/test_gpu_parity.py tests/test_gpu_next.py -x -q -m gpu 2>&1 | tail -2
python tools/tc_probe_c2.py 2>&1 | grep "mode="
for w in c2 c4 c5_cos c3_e8; do
  timeout 300 python bench.py --workload $w 2>/dev/null | tail -1 > gpurun_out/at_$w.json
  python -c "import json;d=json.load(open('gpurun_out/at_$w.json'));print('$w', round(d['ms_per_step'],4), d['step_ms_stats'], d['roofline']['frac'], d['roofline'].get('kernel_ms'), d['breakdown_ms'])"
done
