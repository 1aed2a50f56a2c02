"""One C4 machine step with direct batches (W8 E8 M512) for an ncu launch
list of the batch kernels (k_launch_gather_edge)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402

res, _ = run_native(32768, 1, workers=8, executors=8, max_agg=512, zero_copy=4)
print(res.step_ms)
