"""C4 direct batches at larger aggregation widths: POLLING vs FENCE (events
and words) at 8 and 16 workers, median of 3 interleaved runs."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

P, F = IntegrationMode.POLLING, IntegrationMode.FENCE
for W, E, M in ((8, 8, 512), (8, 8, 1024), (16, 16, 1024), (8, 16, 1024), (4, 8, 1024)):
    ms = {}
    for _ in range(3):
        for comp in ("events", "words"):
            for mode in (P, F):
                res, _ = run_native(32768, 5, workers=W, executors=E, max_agg=M, mode=mode,
                                    zero_copy=4, completion=comp)
                ms.setdefault(f"{comp}_{mode.value}", []).append(statistics.fmean(res.step_ms[1:]))
    med = {k: round(statistics.median(v), 2) for k, v in ms.items()}
    print(json.dumps({"W": W, "E": E, "M": M, **med,
                      "sp_events": round(med["events_fence"] / med["events_polling"], 3),
                      "sp_words": round(med["words_fence"] / med["words_polling"], 3)}), flush=True)
