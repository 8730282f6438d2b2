#!/bin/bash
# ncu --set full (L2 / stall metrics) of the C5 L1 side passes: the thermometer prep, the row-union
# emission, one radix scatter pass; and of one pruned C3 eps=8 and one C5 cosine contraction launch
mkdir -p gpurun_out
for k in k_l1t_prep k_row_pairs k_rs_scatter k_rs_hist k_prep_f32 k_compact k_resolve; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^${k}" --launch-skip 2 --launch-count 1 \
    -o gpurun_out/cf_ncu_$k -f python tools/one_cover.py c5_l1 1 > gpurun_out/cf_ncu_$k.log 2>&1
  python tools/ncu_summary.py gpurun_out/cf_ncu_$k.ncu-rep > gpurun_out/cf_ncu_$k.txt 2>&1; head -40 gpurun_out/cf_ncu_$k.txt
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_tc$" --launch-skip 30 --launch-count 1 \
   -o gpurun_out/cf_ncu_c3e8_member -f python tools/one_cover.py c3_e8 1 > gpurun_out/cf_ncu_c3.log 2>&1
python tools/ncu_summary.py gpurun_out/cf_ncu_c3e8_member.ncu-rep > gpurun_out/cf_ncu_c3e8_member.txt 2>&1; head -30 gpurun_out/cf_ncu_c3e8_member.txt
