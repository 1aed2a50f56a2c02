#!/bin/bash
# Round-end evidence refresh: GPU test suite, smoke, profiles (launch list +
# ncu captures of every hot kernel), star step, default + reference bench.
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
bash scripts/gpu_profiles.sh > gpurun_out/profiles.log 2>&1
timeout 600 python scripts/bench_star.py 5 10 > gpurun_out/star_L5.json 2>&1; tail -c 600 gpurun_out/star_L5.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/star_launches.csv python scripts/bench_star.py 5 2 > /dev/null 2>&1
ls gpurun_out
