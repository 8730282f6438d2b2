#!/bin/bash
# A/B: flat pair emission + 16-byte loads in the unique pass vs the closing-refresh build
mkdir -p gpurun_out/z6
for lib in abtmp/lib_zf.so paper_2601_01405_b200/libbm_b200.so; do
  for w in c3_e8 c5_l1; do
    BM_LIB_PATH=$lib timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline > gpurun_out/z6/b.json 2> gpurun_out/z6/b.err
    python -c "
import json; d=json.load(open('gpurun_out/z6/b.json'))
print('$lib $w', round(d['ms_per_step'],3), d['breakdown_ms'], d['config']['L'], d['config']['M'], d['config']['E'])" || tail -3 gpurun_out/z6/b.err
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/z6/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/z6/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z6/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/z6/launches_c3_e8.csv python tools/one_cover.py c3_e8 1 > gpurun_out/z6/ncu.log 2>&1
python tools/launch_summary.py gpurun_out/z6/launches_c3_e8.csv > gpurun_out/z6/launches_c3_e8.txt 2>&1; head -16 gpurun_out/z6/launches_c3_e8.txt
