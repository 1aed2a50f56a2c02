"""TB_MACHINE_DIAG counters of the bench's C4 machine configuration (direct
batches, W8 E8 M256) with events and with completion words, polling and
fence."""
import os
import statistics
import sys

os.environ["TB_MACHINE_DIAG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

for comp in ("events", "words"):
    for mode in (IntegrationMode.POLLING, IntegrationMode.FENCE):
        res, _ = run_native(32768, 4, mode=mode, completion=comp, **bench.C4_MACHINE)
        sys.stderr.flush()
        print(f"{comp} {mode.value}: {statistics.fmean(res.step_ms[1:]):.2f} ms/step", flush=True)
