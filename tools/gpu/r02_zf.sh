#!/bin/bash
# Round-2 closing refresh: GPU suite, smoke, every bench line (with the oracle baseline),
# the reference arm, the default command's launch list, ncu --set full of the C5 L1 and
# C3 eps=8 contraction launches.
O=gpurun_out/zf; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_c5_l1.json 2> $O/bench_c5_l1.err; echo "bench rc=$?"
for w in c5_cos c3_e8 c3_e4 c3_e2 c4 c2 c1; do
  timeout 900 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 900 python bench.py --impl reference > $O/reference.json 2> $O/reference.err
for w in c5_l1 c5_cos c3_e8 c3_e4 c3_e2 c4 c2 c1; do
  python -c "
import json; d=json.load(open('$O/bench_$w.json'))
print('$w', round(d['ms_per_step'],3), d['breakdown_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['seconds'], 'cpu', (d.get('cpu_baseline') or {}).get('value'))" || tail -3 $O/bench_$w.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tc<" --kernel-name-base demangled \
   --launch-skip 150 --launch-count 1 -o $O/ncu_c5l1_member -f python tools/one_cover.py c5_l1 1 > $O/ncu1.log 2>&1
python tools/ncu_summary.py $O/ncu_c5l1_member.ncu-rep > $O/ncu_c5l1_member.txt 2>&1; head -12 $O/ncu_c5l1_member.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tc<0, 1, 256, 2, 3, 3" --kernel-name-base demangled \
   --launch-skip 30 --launch-count 1 -o $O/ncu_c3e8_member -f python tools/one_cover.py c3_e8 1 > $O/ncu2.log 2>&1
python tools/ncu_summary.py $O/ncu_c3e8_member.ncu-rep > $O/ncu_c3e8_member.txt 2>&1; head -12 $O/ncu_c3e8_member.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv python bench.py --no-cpu-baseline > $O/ncu3.log 2>&1
python tools/launch_summary.py $O/launches_default.csv > $O/launches_default.txt 2>&1; head -12 $O/launches_default.txt
rm -f $O/launches_default.csv
