#!/bin/bash
# two role warps + register cap by __maxnreg__ (no spills) vs the previous build; L1T with 2 or 4 groups
timeout 900 python -m pytest tests/test_gpu_tensor.py -x -q -p no:cacheprovider 2>&1 | tail -1
for v in head r2 r2e4; do
  BM_LIB_PATH=abtmp/lib_$v.so timeout 900 python bench.py --workload c2 --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v c2', round(d['ms_per_step'],4), d['breakdown_ms'].get('member_kernel'))"
  BM_LIB_PATH=abtmp/lib_$v.so timeout 900 python bench.py --workload c3_e8 --steps 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v c3_e8', round(d['ms_per_step'],3), d['breakdown_ms'].get('member_kernel'))"
  BM_LIB_PATH=abtmp/lib_$v.so BM_LOOP_PROFILE=1 timeout 900 python tools/one_cover_path.py c5_cos auto 1 2>&1 | grep "loop profile"
  BM_LIB_PATH=abtmp/lib_$v.so BM_LOOP_PROFILE=1 timeout 900 python tools/one_cover_path.py c5_l1 auto 1 2>&1 | grep "loop profile"
done
