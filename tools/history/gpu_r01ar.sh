#!/bin/bash
# operand row pitch experiment: 16 B multiple vs 128 B atoms
for pad in 0 1; do
  export BM_TC_ROWPAD=$pad
  echo "== BM_TC_ROWPAD=$pad"
  python tools/tc_probe_c2.py 2>&1 | grep -v "trace start\|prologue\|pdl "
  for w in c2 c4 c5_cos c3_e8; do
    timeout 300 python bench.py --workload $w 2>/dev/null | tail -1 > gpurun_out/ar_${w}_$pad.json
    python -c "import json;d=json.load(open('gpurun_out/ar_${w}_$pad.json'));print('$w', round(d['ms_per_step'],4), d['step_ms_stats'], d['roofline']['frac'], d['roofline'].get('kernel_ms'))"
  done
done
