#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_star.py tests/test_gpu_hydro.py -x -q 2>&1 | tail -8
for L in 3 4 5; do timeout 300 python scripts/bench_star.py $L 10 > gpurun_out/star_L$L.json 2>&1; cat gpurun_out/star_L$L.json; done
