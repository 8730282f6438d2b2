#!/bin/bash
# Same-box A/B of library builds: tools/ab_libs.sh "libA libB ..." "w1 w2 ..." [steps]
# (each lib = abtmp/lib_<name>.so; runs interleaved A B A B)
LIBS=$1; WS=$2; ST=${3:-5}
for w in $WS; do
  for rep in 1 2; do
    for l in $LIBS; do
      BM_LIB_PATH=abtmp/lib_$l.so timeout 900 python bench.py --workload $w --steps $ST --no-cpu-baseline 2>/dev/null > gpurun_out/ab_${w}_${l}_$rep.json
      python -c "import json;d=json.load(open('gpurun_out/ab_${w}_${l}_$rep.json'));print('$w $l rep$rep', round(d['ms_per_step'],4), 'kernel', d['roofline']['kernel_ms'], 'bd', d['breakdown_ms'])"
    done
  done
done
