"""C4 machine (W8 E8 M512, direct) with the reference's injected barriers
elided or not (the paper's barrier elision), POLLING / FENCE, events / words,
median of 3 interleaved runs."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

P, F = IntegrationMode.POLLING, IntegrationMode.FENCE
for elide in (False, True):
    ms = {}
    for _ in range(3):
        for comp in ("events", "words"):
            for mode in (P, F):
                res, _ = run_native(32768, 5, workers=8, executors=8, max_agg=512, mode=mode,
                                    zero_copy=4, completion=comp, barrier_elision=elide)
                ms.setdefault(f"{comp}_{mode.value}", []).append(statistics.fmean(res.step_ms[1:]))
    med = {k: round(statistics.median(v), 2) for k, v in ms.items()}
    print(json.dumps({"elision": elide, **med,
                      "sp_events": round(med["events_fence"] / med["events_polling"], 3),
                      "sp_words": round(med["words_fence"] / med["words_polling"], 3)}), flush=True)
