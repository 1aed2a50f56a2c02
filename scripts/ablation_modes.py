"""Polling vs host task vs fence on the native machine across batch-copy
strategies (zero_copy 0 staged / 1 in place / 2 gather / 3 resident): median
of `reps` runs of the mean step time over steps 2..N."""
import json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode
from paper_2303_08058_b200.native_machine import run_native

S = int(sys.argv[1]) if len(sys.argv) > 1 else 512
W, E, M = (int(x) for x in (sys.argv[2:5] if len(sys.argv) > 4 else (8, 32, 8)))
steps, reps = 6, 5
out = {"subgrids": S, "W": W, "E": E, "M": M}
for zc in (0, 1, 2, 3):
    row = {}
    for mode in (IntegrationMode.POLLING, IntegrationMode.HOSTTASK, IntegrationMode.FENCE):
        ms = []
        for _ in range(reps):
            res, _ = run_native(S, steps, workers=W, executors=E, max_agg=M, mode=mode,
                                zero_copy=zc)
            ms.append(statistics.fmean(res.step_ms[1:]))
        row[mode.value] = round(statistics.median(ms), 3)
    row["fence/polling"] = round(row["fence"] / row["polling"], 3)
    out[f"zc{zc}"] = row
print(json.dumps(out))
