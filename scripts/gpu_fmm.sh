#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fmm.py -x -q 2>&1 | tail -15
for L in 3 4 5; do timeout 300 python scripts/bench_fmm.py $L 20 > gpurun_out/fmm_L$L.json 2>&1; cat gpurun_out/fmm_L$L.json; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fmm_m2l -s 3 -c 1 -o gpurun_out/prof_fmm_m2l python scripts/bench_fmm.py 4 1 > gpurun_out/ncu_fmm_m2l.log 2>&1; tail -2 gpurun_out/ncu_fmm_m2l.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fmm_leaf -s 3 -c 1 -o gpurun_out/prof_fmm_leaf python scripts/bench_fmm.py 4 1 > gpurun_out/ncu_fmm_leaf.log 2>&1; tail -2 gpurun_out/ncu_fmm_leaf.log
