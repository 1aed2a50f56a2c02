#!/bin/bash
# Per-kernel table of the max_level-5 star step (ncu launch list) + the step timing.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/star_launches.csv python scripts/bench_star.py 5 2 > gpurun_out/star_ncu.log 2>&1
python scripts/star_kernel_table.py gpurun_out/star_launches.csv > gpurun_out/star_kernels.txt 2>&1
head -16 gpurun_out/star_kernels.txt
timeout 300 python scripts/bench_star.py 5 10
