#!/bin/bash
# L1T wait trace / timeline at HEAD (diagnostic build) + C3 launch list
mkdir -p gpurun_out/z3
W=abtmp/lib_wtrace.so
BM_LIB_PATH=$W BM_TC_TRACE=2 timeout 600 python tools/one_cover.py c5_l1 1 2> gpurun_out/z3/wtrace.log | tail -1
grep wtrace gpurun_out/z3/wtrace.log | sed -n '150p;151p;152p'
BM_LIB_PATH=$W BM_TC_TRACE=3 timeout 600 python tools/one_cover.py c5_l1 1 2> gpurun_out/z3/tline.log | tail -1
grep tline gpurun_out/z3/tline.log | sed -n '150p;151p;152p'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/z3/launches_c3_e8.csv python tools/one_cover.py c3_e8 1 > gpurun_out/z3/ncu.log 2>&1
python tools/launch_summary.py gpurun_out/z3/launches_c3_e8.csv > gpurun_out/z3/launches_c3_e8.txt 2>&1; head -40 gpurun_out/z3/launches_c3_e8.txt
BM_PRUNE_TRACE=1 timeout 600 python bench.py --workload c3_e8 --steps 5 --no-cpu-baseline > gpurun_out/z3/b.json 2> gpurun_out/z3/b.err
python -c "
import json; d=json.load(open('gpurun_out/z3/b.json'))
print('c3_e8', round(d['ms_per_step'],3), d['breakdown_ms'], d['config']['L'], d['config']['M'], d['config']['E'])" || tail -3 gpurun_out/z3/b.err
grep prune gpurun_out/z3/b.err | tail -6
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "prun or fullsize or fps" > gpurun_out/z3/pytest_sub.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/z3/pytest_sub.log
