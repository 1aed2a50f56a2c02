"""Native machine: reference op sequence (H2D ; kernel ; D2H per batch) vs
zero-copy batches (the kernel in place on the pinned staging buffer), in
every completion mode. Median of 3 runs of the mean step time (steps 2..N).
usage: python scripts/zero_copy_ablation.py [subgrids] [steps]"""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    out = {"config": f"native machine, {S} sub-grids x {steps} steps, 8 workers, "
                     "32 executors, max 8, median of 3"}
    sums = set()
    for zc in (False, True):
        for mode in (IntegrationMode.POLLING, IntegrationMode.HOSTTASK, IntegrationMode.FENCE):
            ms = []
            for _ in range(3):
                res, _ = run_native(S, steps, workers=8, executors=32, max_agg=8, mode=mode,
                                    zero_copy=zc)
                ms.append(statistics.fmean(res.step_ms[1:]))
                sums.add(res.checksum.hex())
            out[f"{'zero_copy' if zc else 'staged'}_{mode.value}_ms"] = statistics.median(ms)
    out["checksums_identical"] = len(sums) == 1
    print(json.dumps(out))


if __name__ == "__main__":
    main()
