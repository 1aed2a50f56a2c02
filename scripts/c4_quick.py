"""C4 machine quick timing: W8 E8 M512 direct, POLLING / FENCE with events,
median of 3 interleaved runs (mean of steps 2..5)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

ms = {}
for _ in range(3):
    for mode in (IntegrationMode.POLLING, IntegrationMode.FENCE):
        res, _ = run_native(32768, 5, workers=8, executors=8, max_agg=512, mode=mode, zero_copy=4)
        ms.setdefault(mode.value, []).append(statistics.fmean(res.step_ms[1:]))
print(json.dumps({k: round(statistics.median(v), 3) for k, v in ms.items()}))
