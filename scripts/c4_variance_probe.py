"""Run-to-run variance of the C4 machine (resident, M256): every run's mean
step time (steps 2..5) for POLLING and FENCE interleaved, by (workers,
executors); argv: repeats."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 5
if os.environ.get("PROBE_IMPORT"):     # e.g. "torch" or "bench": the bench's process context
    print("affinity before import", len(os.sched_getaffinity(0)), flush=True)
    __import__(os.environ["PROBE_IMPORT"])
    print("affinity after import", len(os.sched_getaffinity(0)), "threads",
          len(os.listdir("/proc/self/task")), flush=True)
for W, E in ((16, 8), (16, 16)):
    ms = {"polling": [], "fence": []}
    for _ in range(R):
        for mode in (IntegrationMode.POLLING, IntegrationMode.FENCE):
            res, _ = run_native(32768, 5, workers=W, executors=E, max_agg=256, mode=mode,
                                zero_copy=3)
            ms[mode.value].append(round(statistics.fmean(res.step_ms[1:]), 2))
    print(json.dumps({"W": W, "E": E, "pin": os.environ.get("TB_PIN_WORKERS", "0"), **ms,
                      "median_speedup": round(statistics.median(ms["fence"])
                                              / statistics.median(ms["polling"]), 3)}),
          flush=True)
