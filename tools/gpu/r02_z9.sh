#!/bin/bash
# A/B: 32 slices per cell in the centre / radius passes vs 8; then the GPU suite and smoke on the new build
O=gpurun_out/z9; mkdir -p $O
for lib in abtmp/lib_z8.so paper_2601_01405_b200/libbm_b200.so; do
  BM_LIB_PATH=$lib BM_PRUNE_TRACE=1 timeout 600 python bench.py --workload c3_e8 --steps 5 --no-cpu-baseline > $O/b.json 2> $O/b.err
  python -c "
import json; d=json.load(open('$O/b.json'))
print('$lib c3_e8', round(d['ms_per_step'],3), d['breakdown_ms'], d['config']['L'], d['config']['M'], d['config']['E'])" || tail -3 $O/b.err
  grep "prune stats" $O/b.err | tail -1
done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
