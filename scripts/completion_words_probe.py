"""Completion by events vs by kernel-stored words (native machine, direct
batches), POLLING and FENCE interleaved, median of 3 (mean of steps 2..N):
C4 at (W, E) = (16, 8), (8, 8), (16, 16) with M256; the paper's 512 scenario
E32 M8 at 2/4/8 workers; and the API-bound point M1, 16 workers, E16 / E128."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

P, F = IntegrationMode.POLLING, IntegrationMode.FENCE
cases = [("C4", 32768, 5, dict(workers=w, executors=e, max_agg=256))
         for w, e in ((16, 8), (8, 8), (16, 16))]
cases += [("512", 512, 8, dict(workers=w, executors=32, max_agg=8)) for w in (2, 4, 8)]
cases += [("512_M1", 512, 6, dict(workers=16, executors=e, max_agg=1)) for e in (16, 128)]
for name, S, steps, kw in cases:
    ms = {}
    for _ in range(3):
        for comp in ("events", "words"):
            for mode in (P, F):
                res, _ = run_native(S, steps, mode=mode, zero_copy=4, completion=comp, **kw)
                ms.setdefault(f"{comp}_{mode.value}", []).append(
                    round(statistics.fmean(res.step_ms[1:]), 3))
    med = {k: statistics.median(v) for k, v in ms.items()}
    print(json.dumps({"case": name, **kw, **{k: round(v, 3) for k, v in med.items()},
                      "speedup_events": round(med["events_fence"] / med["events_polling"], 3),
                      "speedup_words": round(med["words_fence"] / med["words_polling"], 3),
                      "words_polling_vs_events_fence": round(med["events_fence"]
                                                             / med["words_polling"], 3)}),
          flush=True)
