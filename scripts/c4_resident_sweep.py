"""C4 (32768 sub-grids, reference task structure) on the native machine,
resident batches: step ms by (workers, executors) for POLLING and FENCE
(M = 256), two runs each; one JSON line per cell."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

for W in (4, 8, 16):
    for E in (8, 16):
        row = {"workers": W, "executors": E, "max_agg": 256, "zero_copy": 3}
        for mode in (IntegrationMode.POLLING, IntegrationMode.FENCE):
            ms = []
            for _ in range(2):
                res, _ = run_native(32768, 4, workers=W, executors=E, max_agg=256, mode=mode,
                                    zero_copy=3)
                ms.append(statistics.fmean(res.step_ms[1:]))
            row[mode.value + "_ms"] = [round(x, 2) for x in ms]
        row["speedup"] = round(min(row["fence_ms"]) / min(row["polling_ms"]), 3)
        print(json.dumps(row), flush=True)
