#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
python scripts/e2e_timeline.py 32768 16 > gpurun_out/e2e_timeline.jsonl 2>&1; tail -2 gpurun_out/e2e_timeline.jsonl
for c in 8 16 32; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-chunks $c --e2e-steps 20 > gpurun_out/bench_e2e_c$c.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_e2e_c$c.json').read().strip().splitlines()[-1]);print('c$c', d['e2e'])"; done
