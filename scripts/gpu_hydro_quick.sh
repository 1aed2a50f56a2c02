#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hydro.py -x -q 2>&1 | tail -3
for S in 4096 32768; do timeout 300 python scripts/bench_hydro.py $S 20 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($S, round(d['ms'],4), round(d['frac'],3))"; done
