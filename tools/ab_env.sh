#!/bin/bash
# A/B of one environment switch over bench workloads: tools/ab_env.sh VAR "w1 w2 ..." [steps]
VAR=$1; WS=$2; ST=${3:-10}
for w in $WS; do
  for v in 0 1; do
    if [ $v = 0 ]; then E="env -u $VAR"; else E="env $VAR=1"; fi
    $E timeout 900 python bench.py --workload $w --steps $ST --no-cpu-baseline 2>/dev/null > gpurun_out/ab_${w}_$v.json
    python -c "import json;d=json.load(open('gpurun_out/ab_${w}_$v.json'));print('$w $VAR=$v', round(d['ms_per_step'],4), d['step_ms_stats']['median'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
  done
done
