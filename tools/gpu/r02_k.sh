#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2 3; do
for mode in clocks noclocks slow; do
  if [ $mode = noclocks ]; then E="env BM_NO_CLOCKS=1"; elif [ $mode = slow ]; then E="env BM_CLOCK_MS=1000"; else E="env"; fi
  $E timeout 600 python bench.py --workload c3_e2 --steps 10 --no-cpu-baseline > gpurun_out/k_$mode.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k_$mode.json')); print('$mode', round(d['ms_per_step'],2), [round(x,1) for x in d['step_ms_all']])"
done
done
