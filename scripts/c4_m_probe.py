"""C4 direct batches, polling with events / words: step time by (executors,
max_agg) at 8 workers, median of 3."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

for E in (4, 8, 16):
    for M in (128, 256, 512, 1024):
        row = {"E": E, "M": M}
        for comp in ("events", "words"):
            ms = []
            for _ in range(3):
                res, _ = run_native(32768, 5, workers=8, executors=E, max_agg=M,
                                    mode=IntegrationMode.POLLING, zero_copy=4, completion=comp)
                ms.append(statistics.fmean(res.step_ms[1:]))
            row[comp] = round(statistics.median(ms), 2)
            row[comp + "_batch"] = round(res.per_step[-1].mean_batch, 1)
        print(json.dumps(row), flush=True)
