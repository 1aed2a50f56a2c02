#!/bin/bash
# Refresh the committed profiles: launch list of the bench (no ablation / CPU
# leg, which only add host work and tiny machine kernels), one full ncu capture
# of the timed K2 launch per variant, and the default bench line.
set -x
mkdir -p gpurun_out
rm -f gpurun_out/prof_k2_*.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-ablation > gpurun_out/ncu_launch.log 2>&1
for impl in bulk1 bulk reg; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 18 -c 1 -o gpurun_out/prof_k2_$impl python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-ablation --step-impl $impl > gpurun_out/ncu_full_$impl.log 2>&1
done
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 3000 gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2>&1; tail -c 600 gpurun_out/bench_reference.json
