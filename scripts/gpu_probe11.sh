#!/bin/bash
set -x
mkdir -p gpurun_out/nat2
timeout 900 python -m pytest tests/test_gpu_native_machine.py -x -q -s 2>&1 | tail -3
for sw in executors aggregation workers; do
 for mode in polling hosttask; do
  timeout 1200 python -m paper_2303_08058_b200.cli --engine native --subgrids 512 --steps 5 --repeats 3 --sweep $sw --integration $mode > gpurun_out/nat2/sweep_${mode}_${sw}.csv 2>&1; cat gpurun_out/nat2/sweep_${mode}_${sw}.csv
 done
done
for mode in polling hosttask; do
  timeout 900 python -m paper_2303_08058_b200.cli --engine native --subgrids 32768 --steps 3 --repeats 1 --workers 8 --executors 32 --max-agg 8 --integration $mode > gpurun_out/nat2/c4_$mode.csv 2>&1; tail -1 gpurun_out/nat2/c4_$mode.csv
done
for el in on off; do timeout 900 python -m paper_2303_08058_b200.cli --engine native --subgrids 64 --steps 15 --repeats 3 --workers 4 --executors 1 --max-agg 2 --barrier-elision $el > gpurun_out/nat2/elision_$el.csv 2>&1; tail -1 gpurun_out/nat2/elision_$el.csv; done
timeout 600 python bench.py --steps 200 --warmup 10 --cpu-budget 5 > gpurun_out/bench_default.json 2>&1; tail -c 2600 gpurun_out/bench_default.json
