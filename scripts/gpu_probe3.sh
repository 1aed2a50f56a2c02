#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python scripts/e2e_probe.py 32768 > gpurun_out/e2e_probe.json 2>&1; cat gpurun_out/e2e_probe.json
timeout 600 python bench.py --steps 200 --warmup 10 --cpu-budget 5 > gpurun_out/bench_default.json 2>&1; tail -c 2500 gpurun_out/bench_default.json
for mode in polling hosttask; do
 for sw in executors aggregation; do
  timeout 1200 python -m paper_2303_08058_b200.cli --subgrids 512 --steps 4 --repeats 1 --workers 8 --sweep $sw --integration $mode > gpurun_out/sweep_${mode}_${sw}.csv 2> gpurun_out/sweep_${mode}_${sw}.err; cat gpurun_out/sweep_${mode}_${sw}.csv
 done
done
timeout 900 python -m paper_2303_08058_b200.cli --subgrids 512 --steps 4 --repeats 1 --workers 8 --executors 32 --max-agg 8 --switch-interval-us 100 > gpurun_out/sw100.csv 2>&1; cat gpurun_out/sw100.csv
