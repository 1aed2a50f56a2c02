"""C4 (32768 sub-grids, reference task structure) on the native machine in
the resident batch mode (zero_copy = 3) with TB_MACHINE_DIAG counters, per
completion mode; argv: workers executors max_agg."""
import os
import statistics
import sys

os.environ["TB_MACHINE_DIAG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

W, E, M = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (16, 8, 256)))
for mode in IntegrationMode:
    res, _ = run_native(32768, 3, workers=W, executors=E, max_agg=M, mode=mode, zero_copy=3)
    sys.stderr.flush()
    print(f"C4 resident W{W} E{E} M{M} {mode.value}: step_ms={statistics.fmean(res.step_ms[1:]):.3f} "
          f"batch={res.per_step[-1].mean_batch:.1f}", flush=True)
