#!/bin/bash
# lean tf32 epilogue: 4 groups (96 regs) vs 2 groups (168 regs), same box; C5 cosine and C2
for v in base leg2; do
  BM_LIB_PATH=abtmp/lib_$v.so timeout 600 python -m pytest tests/test_gpu_tensor.py -k "cosine" -x -q -p no:cacheprovider 2>&1 | tail -1
  BM_LIB_PATH=abtmp/lib_$v.so BM_LOOP_PROFILE=1 timeout 900 python tools/one_cover_path.py c5_cos auto 2 2>&1 | tail -2
  BM_LIB_PATH=abtmp/lib_$v.so timeout 900 python bench.py --workload c2 --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c2', round(d['ms_per_step'],4), d['breakdown_ms'].get('member_kernel'))"
done
