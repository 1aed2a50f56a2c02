"""K7 FMM gravity benchmark (BASELINE config 3: "FMM multipole+monopole
interaction kernels only, rotating star max_level 4"). Prints one JSON line:
per-kernel times (CUDA events on the launching stream, L2 flushed before each
timed solve), cells/s of the whole solve, and each interaction kernel's FP64
issue rate against the measured FP64 peak (profiles/fp64_peak.json).
Parity unpinned (self-authored oracle, see oracle/fmm_oracle.py)."""

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import fmm_oracle as f  # noqa: E402  (synthetic inputs only)
from paper_2303_08058_b200.gravity import GravitySolver  # noqa: E402

# FP64 thread-instructions per interaction (counted from the kernels):
# M2L: D tensor ~45 + contraction 84 FMA; leaf: 4 FMA per monopole partner.
M2L_INSTR, LEAF_INSTR = 129, 4


def interactions(L):
    """Interactions the kernels execute: (M2L over levels 0..L-1, leaf).
    Off-domain partners are computed too (zero mass), so per-target counts
    depend only on the child octant; level 0 is counted exactly."""
    import numpy as np
    per = 0
    for o in f.CHILD:
        for P in f.PNEAR:
            for c in f.CHILD:
                q = [o[a] - 2 * P[a] - c[a] for a in range(3)]
                per += sum(x * x for x in q) > 4
    m2l = sum((8 << lev) ** 3 * per // 8 for lev in range(1, L))
    g = np.stack(np.meshgrid(*[np.arange(8)] * 3, indexing="ij")).reshape(3, -1)
    d = g[:, :, None] - g[:, None, :]
    m2l += int(((d * d).sum(0) > 4).sum())
    return m2l, (8 << L) ** 3 * 264


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    rho = torch.from_numpy(f.rotating_star_density(L)).cuda()
    s = GravitySolver(L)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        s.solve(rho)
    names = ["upward", "m2l", "downward", "leaf"]
    tot = {k: 0.0 for k in names + ["solve"]}
    torch.cuda.synchronize()
    for _ in range(reps):
        flush.fill_(1)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        s.upward(rho)
        ev[1].record()
        s.m2l()
        ev[2].record()
        s.downward()
        ev[3].record()
        s.leaf(rho)
        ev[4].record()
        torch.cuda.synchronize()
        for i, k in enumerate(names):
            tot[k] += ev[i].elapsed_time(ev[i + 1])
        tot["solve"] += ev[0].elapsed_time(ev[4])
    ms = {k: v / reps for k, v in tot.items()}
    try:
        peak = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["dfma_instr_per_s"]
        src = "profiles/fp64_peak.json (tb_fp64_probe)"
    except Exception:  # noqa: BLE001
        peak, src = 64 * 148 * 1.965e9, "nominal 64/clk/SM x 148 x 1965 MHz"
    nm, nl = interactions(L)
    cells = (8 << L) ** 3
    rate_m2l = nm * M2L_INSTR / (ms["m2l"] * 1e-3)
    rate_leaf = nl * LEAF_INSTR / (ms["leaf"] * 1e-3)
    print(json.dumps({
        "workload": f"FMM gravity, rotating star, max_level {L} ({cells} leaf cells)",
        "ms": ms, "cells_per_s": cells / (ms["solve"] * 1e-3),
        "m2l_interactions": nm, "leaf_interactions": nl,
        "m2l_fp64_instr_per_s": rate_m2l, "m2l_fp64_frac": rate_m2l / peak,
        "leaf_fp64_instr_per_s": rate_leaf, "leaf_fp64_frac": rate_leaf / peak,
        "fp64_peak_instr_per_s": peak, "peak_source": src,
        "l2": "flushed before every timed solve",
        "parity": "unpinned (self-authored oracle; 1e-10 relative)"}))


if __name__ == "__main__":
    main()
