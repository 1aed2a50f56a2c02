#!/bin/bash
# The paper's sweeps on the native machine with zero-copy batches (run under
# gpurun); CSV rows (the reference harness's columns) land in
# gpurun_out/native_zc/*.csv. Each row's speedup_vs_fence is against the
# fence twin of the same zero-copy configuration.
O=gpurun_out/native_zc; mkdir -p $O
CLI="python -m paper_2303_08058_b200.cli --engine native --zero-copy on"
for mode in polling hosttask; do
  for sw in executors aggregation; do
    timeout 900 $CLI --subgrids 512 --steps 5 --repeats 3 --workers 8 --sweep $sw --integration $mode > $O/sweep_${mode}_${sw}.csv 2>> $O/err.log
  done
done
timeout 900 $CLI --subgrids 512 --steps 5 --repeats 3 --executors 32 --max-agg 8 --sweep workers > $O/sweep_polling_workers.csv 2>> $O/err.log
timeout 1500 $CLI --subgrids 32768 --steps 2 --repeats 1 --workers 8 --executors 32 --max-agg 8 > $O/c4_polling.csv 2>> $O/err.log
tail -n +1 $O/*.csv
