#!/bin/bash
# Quick GPU check: smoke, the GPU test suite, hydro bench, default bench line.
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -25
timeout 300 python scripts/bench_hydro.py 4096 50 > gpurun_out/hydro.json 2>&1; cat gpurun_out/hydro.json
timeout 300 python scripts/bench_hydro.py 32768 20 > gpurun_out/hydro_c4.json 2>&1; cat gpurun_out/hydro_c4.json
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 3000 gpurun_out/bench_default.json
