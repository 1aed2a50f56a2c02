#!/bin/bash
set -x
mkdir -p gpurun_out
python scripts/e2e_probe.py 32768 16 > gpurun_out/e2e_probe.json 2>&1; cat gpurun_out/e2e_probe.json
python scripts/e2e_probe.py 32768 4 > gpurun_out/e2e_probe4.json 2>&1; cat gpurun_out/e2e_probe4.json
for impl in reg bulk; do
  timeout 600 python bench.py --workload c5 --steps 50 --warmup 5 --no-cpu-baseline --step-impl $impl --e2e-steps 3 > gpurun_out/bench_c5_$impl.json 2>&1; tail -c 900 gpurun_out/bench_c5_$impl.json; echo
done
for cfg in "--workers 4 --executors 1 --max-agg 8" "--workers 8 --executors 1 --max-agg 32" "--workers 8 --executors 32 --max-agg 8" "--workers 8 --executors 32 --max-agg 1"; do
  timeout 900 python -m paper_2303_08058_b200.cli --subgrids 64 --steps 15 --repeats 3 $cfg --integration polling >> gpurun_out/ablation64.csv 2>> gpurun_out/ablation64.err
  timeout 900 python -m paper_2303_08058_b200.cli --subgrids 64 --steps 15 --repeats 3 $cfg --integration hosttask >> gpurun_out/ablation64.csv 2>> gpurun_out/ablation64.err
done
cat gpurun_out/ablation64.csv; tail -3 gpurun_out/ablation64.err
