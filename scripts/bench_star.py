"""Coupled rotating-star step (hydro K6 + FMM gravity K7 + SSP-RK2) per-step
time at max_level L, eager and CUDA-graph replay. One JSON line. Parity
unpinned (oracle/star_oracle.py)."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.star import RotatingStarStep  # noqa: E402


def timed(st, steps, graph):
    for _ in range(3):
        st.step(graph=graph)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        st.step(graph=graph)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    concurrent = not (len(sys.argv) > 3 and sys.argv[3] == "serial")
    st = RotatingStarStep(L, concurrent=concurrent)
    m0, _, e0 = st.totals()
    eager = timed(st, steps, False)
    graph = timed(st, steps, True)
    m1, p1, e1 = st.totals()
    cells = st.n ** 3
    print(json.dumps({
        "workload": f"rotating star step (hydro + FMM gravity, SSP-RK2), max_level {L}, "
                    f"{cells} cells",
        "hydro_branch": "side stream" if concurrent else "serial",
        "ms_per_step_eager": eager, "ms_per_step_graph": graph,
        "cells_per_s": cells / (min(eager, graph) * 1e-3),
        "launches_per_step": st.launches_per_step(),
        "mass_rel_drift": abs(m1 - m0) / m0, "momentum": p1, "energy_rel_change": (e1 - e0) / e0,
        "l2": f"state {5 * cells * 8 / 2**20:.0f} MiB, steps back to back",
        "parity": "unpinned (self-authored spec oracle/star_oracle.py; 1e-10 per cell)"}))


if __name__ == "__main__":
    main()
