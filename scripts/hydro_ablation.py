"""Polling vs host-task vs fence on the native machine running the hydro
kernel (the paper's experiment shape: PAPER.md:762-782 — per-sub-grid hydro
tasks with aggregated launches; 32 executors x max 8 aggregated, 8 workers,
PAPER.md:931-933). One JSON line per size. Parity unpinned (oracle/hydro_oracle.py)."""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.hydro import rotating_star  # noqa: E402
from paper_2303_08058_b200.native_machine import run_native_hydro  # noqa: E402


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [512, 4096]
    for S in sizes:
        I, _ = rotating_star(S)
        I = I.numpy()
        steps = 8 if S <= 4096 else 4
        row = {"subgrids": S, "cells": S * 512, "workers": 8, "executors": 32, "max_agg": 8,
               "steps": steps}
        for mode in IntegrationMode:
            ms, sig = [], set()
            for _ in range(3):
                per, U = run_native_hydro(I, steps, workers=8, executors=32, max_agg=8,
                                          mode=mode, task_subgrids=1 if S <= 4096 else 8)
                ms.append(statistics.fmean(m.wall_ms for m in per[2:]))   # 2 warm-up steps
                sig.add(U.tobytes().__hash__())
            row[f"{mode.value}_ms_per_step"] = statistics.median(ms)
            row[f"{mode.value}_mean_batch"] = per[-1].mean_batch
            row[f"{mode.value}_launches_per_step"] = per[-1].launches
            row[f"{mode.value}_deterministic"] = len(sig) == 1
        row["speedup_polling_vs_fence"] = row["fence_ms_per_step"] / row["polling_ms_per_step"]
        row["speedup_hosttask_vs_fence"] = row["fence_ms_per_step"] / row["hosttask_ms_per_step"]
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
