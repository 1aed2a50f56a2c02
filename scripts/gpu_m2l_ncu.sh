#!/bin/bash
# ncu --set full (source counters) of the M2L and leaf kernels at max_level 4 (config 3).
mkdir -p gpurun_out/k7
rm -f gpurun_out/k7/*.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fmm_m2l|k_fmm_leaf_mma" -s 2 -c 2 -o gpurun_out/k7/prof python scripts/bench_fmm.py 4 2 > gpurun_out/k7/ncu.log 2>&1
tail -3 gpurun_out/k7/ncu.log
