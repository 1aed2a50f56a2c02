#!/bin/bash
# Round-2 evidence: launch list of the bench's data path, one full ncu capture
# of K2 (k_step_bulk, integer-pipe min) and K6 (variant 508), the back-to-back
# K2 DRAM traffic, two driver-command bench lines and the reference arm.
set -x
mkdir -p gpurun_out/r02
rm -f gpurun_out/r02/*.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches.csv python bench.py --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-ablation --no-kernels > gpurun_out/r02/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 40 -c 1 -o gpurun_out/r02/prof_k2 python bench.py --steps 2 --warmup 5 --warm-ms 0 --e2e-steps 0 --no-cpu-baseline --no-ablation --no-kernels > gpurun_out/r02/ncu_full_k2.log 2>&1
timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:k_step -s 20 -c 3 python scripts/k2_b2b.py > gpurun_out/r02/k2_b2b.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hydro -s 3 -c 1 -o gpurun_out/r02/prof_hydro python scripts/bench_hydro.py 4096 2 > gpurun_out/r02/ncu_hydro.log 2>&1
for i in 1 2; do timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02/bench_$i.json 2> gpurun_out/r02/bench_$i.err; done
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02/bench_reference.json 2>&1
tail -c 300 gpurun_out/r02/bench_1.json; tail -c 300 gpurun_out/r02/bench_reference.json
ls gpurun_out/r02
