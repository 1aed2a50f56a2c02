"""C4 direct batches: step time by (workers, executors) for POLLING / FENCE
with events and words, 3 runs each interleaved (medians) — run under
TB_AFFINITY=0/1 and TB_RESUME_CHUNK to compare dealing policies."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

P, F = IntegrationMode.POLLING, IntegrationMode.FENCE
for W, E in ((8, 8), (16, 8), (8, 2), (16, 4)):
    ms = {}
    for _ in range(3):
        for comp in ("events", "words"):
            for mode in (P, F):
                res, _ = run_native(32768, 5, workers=W, executors=E, max_agg=256, mode=mode,
                                    zero_copy=4, completion=comp)
                ms.setdefault(f"{comp}_{mode.value}", []).append(statistics.fmean(res.step_ms[1:]))
    med = {k: round(statistics.median(v), 2) for k, v in ms.items()}
    print(json.dumps({"W": W, "E": E, "affinity": os.environ.get("TB_AFFINITY", "1"),
                      "chunk": os.environ.get("TB_RESUME_CHUNK", "16"), **med}), flush=True)
