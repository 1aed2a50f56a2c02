#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fmm.py -x -q 2>&1 | tail -3
for L in 4 5; do timeout 300 python scripts/bench_fmm.py $L 20 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($L, {k: round(v,4) for k,v in d['ms'].items()})"; done
