#!/bin/bash
# ncu --set full (source counters) of K6 for each TB_HYDRO_VARIANT given, config 2.
mkdir -p gpurun_out/k6
for v in "$@"; do
  rm -f gpurun_out/k6/prof_$v.ncu-rep
  TB_HYDRO_VARIANT=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hydro -s 3 -c 1 -o gpurun_out/k6/prof_$v python scripts/bench_hydro.py 4096 2 > gpurun_out/k6/ncu_$v.log 2>&1
  tail -2 gpurun_out/k6/ncu_$v.log
done
