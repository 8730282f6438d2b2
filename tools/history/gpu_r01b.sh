# ncu --set full captures: C2 membership kernel (CUDA cores), C3 eps=8 prefix tcgen05 contraction
set -x
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_pairsILi0ELi5ELi4ELi2E" -s 1 -c 1 -o gpurun_out/prof_c2_member python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 300 python bench.py --workload c3_e8 --n 200000 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_tc" -s 1 -c 1 -o gpurun_out/prof_c3_tc python bench.py --workload c3_e8 --n 200000 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_c3.log 2>&1; echo "ncu c3 rc=$?"
cat gpurun_out/plain_c3.log
ls -la gpurun_out
