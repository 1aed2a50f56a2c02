#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2 3; do for impl in bulk1 bulk reg; do
  timeout 300 python bench.py --workload c5 --steps 30 --warmup 5 --no-cpu-baseline --no-ablation --step-impl $impl --e2e-steps 1 > gpurun_out/b5_${impl}_$rep.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/b5_${impl}_$rep.json').read().strip().splitlines()[-1]);print('$impl c5', round(d['roofline']['k2_ms']*1e3,1), round(d['roofline']['frac'],4))"
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-ablation --step-impl $impl --e2e-steps 1 > gpurun_out/b4_${impl}_$rep.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/b4_${impl}_$rep.json').read().strip().splitlines()[-1]);print('$impl c4', round(d['roofline']['k2_ms']*1e3,1), round(d['roofline']['frac'],4))"
done; done
