#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "edges or big_tile or full" 2>&1 | tail -1
for w in c4 c5_cos; do
  timeout 900 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/ab_bench_$w.json 2> gpurun_out/ab_bench_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_bench_$w.json'))
print('$w', round(d['ms_per_step'],3), d['breakdown_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['seconds'])" || tail -3 gpurun_out/ab_bench_$w.err
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tc<" --kernel-name-base demangled --launch-skip 4 --launch-count 1 -o gpurun_out/ab_ncu_c4_member -f python tools/one_cover.py c4 1 > gpurun_out/ab_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/ab_ncu_c4_member.ncu-rep 2>&1 | head -24
