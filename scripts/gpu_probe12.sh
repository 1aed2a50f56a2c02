#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
for impl in bulk1 reg; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-ablation --step-impl $impl --e2e-steps 2 > gpurun_out/b_${impl}.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/b_${impl}.json').read().strip().splitlines()[-1]);print('$impl c4', d['roofline']['k2_ms']*1e3, d['roofline']['frac'], d['clocks'])"
  timeout 300 python bench.py --workload c5 --steps 30 --warmup 5 --no-cpu-baseline --no-ablation --step-impl $impl --e2e-steps 1 > gpurun_out/b5_${impl}.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/b5_${impl}.json').read().strip().splitlines()[-1]);print('$impl c5', d['roofline']['k2_ms']*1e3, d['roofline']['frac'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 18 -c 1 -o gpurun_out/prof_k2_bulk1 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-ablation --step-impl bulk1 > gpurun_out/ncu_full_bulk1.log 2>&1
