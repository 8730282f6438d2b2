CMD="python bench.py --workload c5_l1 --n 4000000 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_c5p.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --kernel-name-base function -k "regex:k_compact|k_rs_scatter|k_keys_to_bits|k_bits_csr|k_unique_compact|k_pair_emit|k_prep_f32|k_l1_quantize|k_minmax|k_rs_hist" -s 300 -c 14 -o gpurun_out/prof_c5_hbm $CMD > gpurun_out/ncu_c5hbm.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_c5hbm.log
