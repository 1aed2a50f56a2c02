"""Reference acceptance criteria 4 and 5 (pkg/tests/test_acceptance.py:94-122)
measured on the B200, on the Python machine (the reference-facing stack,
cli engine python) and on the native machine: 64 sub-grids x 15 steps,
median of 3 repeats. Criterion 4: host-task no faster than polling at E=1,
M=32, W=8. Criterion 5: barrier elision faster at E=1, M=2, W=4. One JSON
line per engine."""
import json
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200 import cli  # noqa: E402
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402

for engine in ("native", "python"):
    c4 = cli.RunConfig(subgrids=64, steps=15, repeats=3, executors=1, max_agg=32, workers=8,
                       engine=engine)
    ht = cli.run_cell(replace(c4, integration=IntegrationMode.HOSTTASK))
    po = cli.run_cell(replace(c4, integration=IntegrationMode.POLLING))
    c5 = cli.RunConfig(subgrids=64, steps=15, repeats=3, executors=1, max_agg=2, workers=4,
                       engine=engine, inject_barriers=True)
    on = cli.run_cell(replace(c5, barrier_elision=True))
    off = cli.run_cell(replace(c5, barrier_elision=False))
    print(json.dumps({"engine": engine,
                      "c4_hosttask_ms": ht.mean_step_ms, "c4_polling_ms": po.mean_step_ms,
                      "c4_ratio_hosttask_over_polling": ht.mean_step_ms / po.mean_step_ms,
                      "c4_mean_batch": [ht.mean_batch, po.mean_batch],
                      "c5_on_ms": on.mean_step_ms, "c5_off_ms": off.mean_step_ms,
                      "c5_ratio_off_over_on": off.mean_step_ms / on.mean_step_ms,
                      "c5_checksums_equal": on.checksum == off.checksum}), flush=True)
