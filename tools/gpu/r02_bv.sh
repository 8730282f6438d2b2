#!/bin/bash
# round-2 measurement refresh: every bench line (with the oracle baseline), the reference arm,
# the default line's launch list, ncu --set full of one C5 L1 contraction launch
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/bv_smi.txt
timeout 900 python bench.py > gpurun_out/bv_bench_c5_l1.json 2> gpurun_out/bv_bench_c5_l1.err; echo "default rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bv_reference.json 2> gpurun_out/bv_reference.err; echo "ref rc=$?"
for w in c5_cos c3_e8 c3_e4 c3_e2 c4 c2 c1; do
  timeout 900 python bench.py --workload $w --steps 5 > gpurun_out/bv_bench_$w.json 2> gpurun_out/bv_bench_$w.err; echo "$w rc=$?"
done
for f in gpurun_out/bv_bench_*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']
print('$f'.split('bv_bench_')[1], round(d['ms_per_step'],3), 'frac', r['frac'], 'e2e', d['e2e']['seconds'], 'cpu', (d.get('cpu_baseline') or {}).get('value'))"; done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bv_launches_default.csv $CMD > gpurun_out/bv_ncu_launch.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/bv_launches_default.csv > gpurun_out/bv_launches_default.txt 2>&1; head -12 gpurun_out/bv_launches_default.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_tc$" \
   --launch-skip 60 --launch-count 1 -o gpurun_out/bv_ncu_c5l1_member -f python tools/one_cover.py c5_l1 1 > gpurun_out/bv_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/bv_ncu_c5l1_member.ncu-rep > gpurun_out/bv_ncu_c5l1_member.txt 2>&1; head -20 gpurun_out/bv_ncu_c5l1_member.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_tc$" \
   --launch-skip 9 --launch-count 1 -o gpurun_out/bv_ncu_c4_member -f python tools/one_cover.py c4 2 > gpurun_out/bv_ncu4.log 2>&1
python tools/ncu_summary.py gpurun_out/bv_ncu_c4_member.ncu-rep > gpurun_out/bv_ncu_c4_member.txt 2>&1; head -3 gpurun_out/bv_ncu_c4_member.txt
timeout 900 python tools/bench_next.py --reps 3 > gpurun_out/bv_next.jsonl 2> gpurun_out/bv_next.err; echo "next rc=$?"
