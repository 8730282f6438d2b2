#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/aa_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/aa_pytest.log
BM_LIB_PATH=abtmp/lib_rows.so timeout 600 python /tmp/chain.py 100 2>&1 | tail -1 || true
for w in c5_l1 c5_cos c3_e8 c3_e2 c4 c2; do
  timeout 900 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/aa_bench_$w.json 2> gpurun_out/aa_bench_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/aa_bench_$w.json'))
print('$w', round(d['ms_per_step'],3), d['breakdown_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['seconds'])" || tail -3 gpurun_out/aa_bench_$w.err
done
