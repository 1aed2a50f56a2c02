#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 200 --warmup 10 --cpu-budget 5 > gpurun_out/bench_default.json 2>&1; tail -c 1500 gpurun_out/bench_default.json
for impl in reg bulk; do for spw in 1 2 4; do
  timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --step-impl $impl --spw $spw --e2e-steps 2 > gpurun_out/b_${impl}_spw${spw}.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/b_${impl}_spw${spw}.json').read().strip().splitlines()[-1]);print('$impl spw$spw', d['roofline']['k2_ms']*1e3, d['roofline']['frac'])"
done; done
timeout 1500 python -m paper_2303_08058_b200.cli --subgrids 32768 --task-subgrids 64 --steps 2 --repeats 1 --workers 8 --executors 32 --max-agg 8 --integration polling > gpurun_out/c4_abl_poll.csv 2> gpurun_out/c4_abl_poll.err; cat gpurun_out/c4_abl_poll.csv; tail -3 gpurun_out/c4_abl_poll.err
timeout 1500 python -m paper_2303_08058_b200.cli --subgrids 32768 --task-subgrids 64 --steps 2 --repeats 1 --workers 8 --executors 8 --max-agg 4 --integration polling > gpurun_out/c4_abl_poll2.csv 2>&1; cat gpurun_out/c4_abl_poll2.csv
timeout 1500 python -m paper_2303_08058_b200.cli --subgrids 512 --steps 4 --repeats 1 --workers 8 --executors 32 --max-agg 8 --integration polling > gpurun_out/l3_abl_poll.csv 2>&1; cat gpurun_out/l3_abl_poll.csv
