#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_native_machine.py -x -q -s 2>&1 | tail -15
for mode in polling hosttask; do
  timeout 900 python -m paper_2303_08058_b200.cli --engine native --subgrids 512 --steps 5 --repeats 3 --workers 8 --executors 32 --max-agg 8 --integration $mode > gpurun_out/native_512_$mode.csv 2>&1; cat gpurun_out/native_512_$mode.csv
done
timeout 900 python -m paper_2303_08058_b200.cli --engine native --subgrids 32768 --steps 2 --repeats 1 --workers 8 --executors 32 --max-agg 8 > gpurun_out/native_c4.csv 2>&1; cat gpurun_out/native_c4.csv
