"""TB_MACHINE_DIAG counters at the paper's Test-2 graph-1 point that polling
loses: 512 sub-grids, no aggregation (M = 1), 16 workers, E = 16 / 128,
staged batches; POLLING vs FENCE."""
import os
import statistics
import sys

os.environ["TB_MACHINE_DIAG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

for E in (16, 128):
    for mode in (IntegrationMode.POLLING, IntegrationMode.FENCE):
        res, _ = run_native(512, 6, workers=16, executors=E, max_agg=1, mode=mode,
                            zero_copy=int(sys.argv[1]) if len(sys.argv) > 1 else 0)
        sys.stderr.flush()
        print(f"E{E} {mode.value}: {statistics.fmean(res.step_ms[1:]):.2f} ms/step", flush=True)
