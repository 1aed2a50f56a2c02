"""BASELINE config 4 on the native machine (reference task structure: one
task and 15 schedule() calls per sub-grid per step, 32768 sub-grids): step
time by (executors, max_agg, zero-copy mode) for POLLING and its FENCE twin,
to pick the configuration bench.py's ablation.c4 leg runs. One JSON line per
cell; steps 2..N averaged."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

S = 32768
modes = [IntegrationMode.POLLING, IntegrationMode.FENCE]
grid = [(32, 8), (32, 32), (32, 64), (8, 64), (64, 64), (16, 128)]
for zc in (0, 2):
    for e, m in grid:
        row = {"executors": e, "max_agg": m, "zero_copy": zc, "workers": 8}
        for mode in modes:
            res, _ = run_native(S, 3, workers=8, executors=e, max_agg=m, mode=mode, zero_copy=zc)
            row[mode.value + "_ms"] = statistics.fmean(res.step_ms[1:])
            row[mode.value + "_mean_batch"] = res.per_step[-1].mean_batch
        row["speedup"] = row["fence_ms"] / row["polling_ms"]
        print(json.dumps(row), flush=True)
