#!/bin/bash
# Refresh the committed profiles: launch list of the bench's data path, one
# full ncu capture per hot kernel (K2, K6, K7 up/M2L/leaf, star stage), the
# back-to-back K2 DRAM traffic, and the default + reference bench lines.
set -x
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-ablation --no-kernels > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 18 -c 1 -o gpurun_out/prof_k2_bulk1 python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-ablation --no-kernels > gpurun_out/ncu_full_k2.log 2>&1
timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:k_step -s 20 -c 3 python scripts/k2_b2b.py > gpurun_out/k2_b2b.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hydro -s 3 -c 1 -o gpurun_out/prof_hydro python scripts/bench_hydro.py 4096 2 > gpurun_out/ncu_hydro.log 2>&1
for k in m2l leaf; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fmm_$k -s 3 -c 1 -o gpurun_out/prof_fmm_$k python scripts/bench_fmm.py 4 1 > gpurun_out/ncu_fmm_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fmm_up -s 12 -c 1 -o gpurun_out/prof_fmm_up python scripts/bench_fmm.py 4 1 > gpurun_out/ncu_fmm_up.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_star_stage -s 4 -c 1 -o gpurun_out/prof_star_stage python scripts/bench_star.py 4 1 > gpurun_out/ncu_star.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 1500 gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2>&1; tail -c 600 gpurun_out/bench_reference.json
ls gpurun_out
