#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for impl in reg lean pair bulk; do
  timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --step-impl $impl --e2e-steps 2 > gpurun_out/b_${impl}.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/b_${impl}.json').read().strip().splitlines()[-1]);print('$impl c4', d['roofline']['k2_ms']*1e3, d['roofline']['frac'])"
  timeout 300 python bench.py --workload c5 --steps 30 --warmup 5 --no-cpu-baseline --step-impl $impl --e2e-steps 1 > gpurun_out/b5_${impl}.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/b5_${impl}.json').read().strip().splitlines()[-1]);print('$impl c5', d['roofline']['k2_ms']*1e3, d['roofline']['frac'])"
done
for impl in lean pair; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 18 -c 1 -o gpurun_out/prof_k2_$impl python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --step-impl $impl > gpurun_out/ncu_full_$impl.log 2>&1
done
for sw in 5000 1000 100; do
  timeout 900 python -m paper_2303_08058_b200.cli --subgrids 512 --steps 4 --repeats 3 --workers 8 --executors 32 --max-agg 8 --switch-interval-us $sw > gpurun_out/abl512_sw$sw.csv 2>&1; tail -1 gpurun_out/abl512_sw$sw.csv
done
timeout 900 python -m paper_2303_08058_b200.cli --subgrids 64 --steps 15 --repeats 3 --workers 4 --executors 1 --max-agg 8 > gpurun_out/abl64_c3.csv 2>&1; tail -1 gpurun_out/abl64_c3.csv
timeout 900 python -m paper_2303_08058_b200.cli --subgrids 64 --steps 15 --repeats 3 --workers 4 --executors 1 --max-agg 8 --switch-interval-us 100 > gpurun_out/abl64_c3_sw100.csv 2>&1; tail -1 gpurun_out/abl64_c3_sw100.csv
