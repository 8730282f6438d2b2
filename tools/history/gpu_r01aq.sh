#!/bin/bash
# tensor epilogue: d_j prefetch (parity + C2/C3/C4 bench)
timeout 600 python -m pytest tests/test_gpu_tensor.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
for w in c2 c3_e8 c4 c5_cos; do
  timeout 300 python bench.py --workload $w 2>/dev/null | tail -1 > gpurun_out/aq_$w.json
  python -c "import json;d=json.load(open('gpurun_out/aq_$w.json'));print('$w', d['ms_per_step'], d['step_ms_stats'], d['roofline']['frac'], d['roofline'].get('kernel_ms'))"
done
