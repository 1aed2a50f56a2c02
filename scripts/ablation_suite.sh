#!/bin/bash
# The paper's ablations on one B200 (run under gpurun); CSV rows land in
# gpurun_out/ablation/*.csv with the reference harness's columns.
set -x
O=gpurun_out/ablation; mkdir -p $O
CLI="python -m paper_2303_08058_b200.cli"
# Tests 1-2 of the paper: executor and aggregation sweeps,
# 512 sub-grids, polling and host-task each against their fence twin.
for mode in polling hosttask; do
  for sw in executors aggregation; do
    timeout 1200 $CLI --subgrids 512 --steps 4 --repeats 1 --workers 8 --sweep $sw --integration $mode > $O/sweep_${mode}_${sw}.csv 2>> $O/err.log
  done
done
# worker sweep at the paper's best combination (32 executors x 8)
timeout 1200 $CLI --subgrids 512 --steps 4 --repeats 1 --executors 32 --max-agg 8 --sweep workers > $O/sweep_polling_workers.csv 2>> $O/err.log
# Test 3: barrier elision on/off (reference criterion 5 config)
for el in on off; do
  timeout 900 $CLI --subgrids 64 --steps 15 --repeats 3 --workers 4 --executors 1 --max-agg 2 --barrier-elision $el > $O/elision_$el.csv 2>> $O/err.log
done
# event pool on/off
for ep in on off; do
  timeout 900 $CLI --subgrids 512 --steps 4 --repeats 1 --workers 8 --executors 32 --max-agg 8 --event-pool $ep > $O/eventpool_$ep.csv 2>> $O/err.log
done
# C4: max_level 5 = 32768 sub-grids, reference task structure (1 task per
# sub-grid) and coarsened (64 per task)
timeout 1500 $CLI --subgrids 32768 --steps 1 --repeats 1 --warmup-steps 0 --workers 8 --executors 32 --max-agg 8 > $O/c4_tasks1.csv 2>> $O/err.log
timeout 1500 $CLI --subgrids 32768 --task-subgrids 64 --steps 2 --repeats 1 --workers 8 --executors 32 --max-agg 8 > $O/c4_tasks64.csv 2>> $O/err.log
timeout 1500 $CLI --subgrids 32768 --task-subgrids 64 --steps 2 --repeats 1 --workers 8 --executors 32 --max-agg 8 --integration hosttask > $O/c4_tasks64_hosttask.csv 2>> $O/err.log
tail -n +1 $O/*.csv
