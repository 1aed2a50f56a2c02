"""C4 machine: resident (3) vs direct (4) batches, POLLING and FENCE
interleaved, 3 runs each (mean of steps 2..5), W16 E8 M256 and W8 E8."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

for W, E in ((16, 8), (8, 8), (16, 16)):
    ms = {}
    for _ in range(3):
        for zc in (3, 4):
            for mode in (IntegrationMode.POLLING, IntegrationMode.FENCE):
                res, _ = run_native(32768, 5, workers=W, executors=E, max_agg=256, mode=mode,
                                    zero_copy=zc)
                ms.setdefault(f"zc{zc}_{mode.value}", []).append(
                    round(statistics.fmean(res.step_ms[1:]), 2))
    med = {k: statistics.median(v) for k, v in ms.items()}
    print(json.dumps({"W": W, "E": E, **ms,
                      "speedup_zc3": round(med["zc3_fence"] / med["zc3_polling"], 3),
                      "speedup_zc4": round(med["zc4_fence"] / med["zc4_polling"], 3)}), flush=True)
