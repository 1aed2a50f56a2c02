#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
python scripts/e2e_timeline.py 32768 16 > gpurun_out/e2e_timeline.jsonl 2>&1; cat gpurun_out/e2e_timeline.jsonl
python scripts/e2e_timeline.py 32768 8 > gpurun_out/e2e_timeline8.jsonl 2>&1; tail -1 gpurun_out/e2e_timeline8.jsonl
timeout 600 python bench.py --steps 200 --warmup 10 --cpu-budget 5 > gpurun_out/bench_default.json 2>&1; tail -c 1800 gpurun_out/bench_default.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
