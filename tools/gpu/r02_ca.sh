#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "sort or edges or c2 or c1" 2>&1 | tail -1
python tools/sort_bench.py 140000000 39 5
timeout 900 python bench.py --workload c3_e8 --steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c3_e8', round(d['ms_per_step'],3), d['breakdown_ms'])"
