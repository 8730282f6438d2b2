#!/bin/bash
# A/B: cell kernels (Gram-form assign, sliced centre/radius passes, 16-row gather) vs HEAD
mkdir -p gpurun_out/z2
for lib in abtmp/lib_head.so paper_2601_01405_b200/libbm_b200.so; do
  for w in c3_e8 c3_e2; do
    BM_LIB_PATH=$lib BM_PRUNE_TRACE=1 timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/z2/b.json 2> gpurun_out/z2/b.err
    python -c "
import json; d=json.load(open('gpurun_out/z2/b.json'))
print('$lib $w', round(d['ms_per_step'],3), d['breakdown_ms'], d['config']['L'], d['config']['M'], d['config']['E'])" || tail -3 gpurun_out/z2/b.err
    grep prune gpurun_out/z2/b.err | tail -6
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/z2/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/z2/pytest_gpu.log
