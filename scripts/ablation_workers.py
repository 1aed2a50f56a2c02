"""The paper's third ablation graph: the best (E, M)
combination with fewer and fewer workers — polling vs fence vs host task on
the native machine, staged batches (the reference op sequence)."""
import json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode
from paper_2303_08058_b200.native_machine import run_native

S = int(sys.argv[1]) if len(sys.argv) > 1 else 512
zc = int(sys.argv[2]) if len(sys.argv) > 2 else 0
E, M, steps, reps = 32, 8, 6, 5
out = {"subgrids": S, "E": E, "M": M, "zero_copy": zc}
for W in (1, 2, 4, 8, 16):
    row = {}
    for mode in (IntegrationMode.POLLING, IntegrationMode.HOSTTASK, IntegrationMode.FENCE):
        ms = []
        for _ in range(reps):
            res, _ = run_native(S, steps, workers=W, executors=E, max_agg=M, mode=mode,
                                zero_copy=zc)
            ms.append(statistics.fmean(res.step_ms[1:]))
        row[mode.value] = round(statistics.median(ms), 3)
    row["fence/polling"] = round(row["fence"] / row["polling"], 3)
    out[f"W{W}"] = row
print(json.dumps(out))
