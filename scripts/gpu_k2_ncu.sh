#!/bin/bash
# ncu --set full (source counters) of one mid-run K2 launch at the default workload (C4).
mkdir -p gpurun_out/k2
rm -f gpurun_out/k2/*.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 30 -c 1 -o gpurun_out/k2/prof python bench.py --steps 20 --warmup 10 --warm-ms 0 --e2e-steps 0 --no-cpu-baseline --no-ablation --no-kernels > gpurun_out/k2/ncu.log 2>&1
tail -2 gpurun_out/k2/ncu.log
