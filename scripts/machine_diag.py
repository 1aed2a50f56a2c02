"""Native machine host-side diagnostics (TB_MACHINE_DIAG=1 counters on
stderr): the 512 scenario (32 executors, max 8, staged) at 2/4/8 workers and
C4 (bench.C4_MACHINE), POLLING vs FENCE, one run each, mean step ms."""
import os
import statistics
import sys

os.environ["TB_MACHINE_DIAG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

cases = [(512, 6, dict(workers=W, executors=32, max_agg=8, zero_copy=0)) for W in (2, 4, 8)]
cases.append((32768, 3, bench.C4_MACHINE))
for S, steps, kw in cases:
    for mode in (IntegrationMode.POLLING, IntegrationMode.FENCE):
        for rep in range(2):
            res, _ = run_native(S, steps, mode=mode, **kw)
            sys.stderr.flush()
            print(f"S={S} {kw} {mode.value} rep{rep}: step_ms={statistics.fmean(res.step_ms[1:]):.3f} "
                  f"batch={res.per_step[-1].mean_batch:.1f}", flush=True)
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
