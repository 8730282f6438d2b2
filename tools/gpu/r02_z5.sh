#!/bin/bash
# A/B: L1T tail K steps as 32-byte sub-atoms, at 9 / 10 / 11 K steps
mkdir -p gpurun_out/z5
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "l1 or L1" > gpurun_out/z5/pytest_l1.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/z5/pytest_l1.log
for lib in paper_2601_01405_b200/libbm_b200.so abtmp/lib_tail282.so abtmp/lib_tail342.so; do
  BM_LIB_PATH=$lib timeout 600 python bench.py --workload c5_l1 --steps 3 --no-cpu-baseline > gpurun_out/z5/b.json 2> gpurun_out/z5/b.err
  python -c "
import json; d=json.load(open('gpurun_out/z5/b.json'))
print('$lib', round(d['ms_per_step'],3), d['breakdown_ms'], d['config']['L'], d['config']['M'], d['config']['E'], d['greedy'])" || tail -3 gpurun_out/z5/b.err
done
