"""Gather-batch native machine at BASELINE config 4 (reference task
structure, POLLING): step time by workers x executors x max_agg, to pick the
plugin path's configuration. One JSON line per cell (mean of steps 2..3)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

for w in (8, 12, 16):
    for e in (8, 16, 32):
        for m in (64, 128, 256):
            res, _ = run_native(32768, 3, workers=w, executors=e, max_agg=m, zero_copy=2)
            print(json.dumps({"workers": w, "executors": e, "max_agg": m,
                              "polling_ms": statistics.fmean(res.step_ms[1:]),
                              "mean_batch": res.per_step[-1].mean_batch}), flush=True)
