#!/bin/bash
set -x
mkdir -p gpurun_out
python scripts/fp64_probe.py > gpurun_out/fp64_peak.json 2>&1; cat gpurun_out/fp64_peak.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hydro -s 3 -c 1 -o gpurun_out/prof_hydro python scripts/bench_hydro.py 4096 2 > gpurun_out/ncu_hydro.log 2>&1; tail -3 gpurun_out/ncu_hydro.log
