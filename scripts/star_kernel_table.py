"""Per-kernel roofline table of one rotating-star step at max_level 5 from an
ncu launch list (gpu__time_duration.sum, --clock-control none) of
`scripts/bench_star.py 5 2`: median duration per kernel launch against the
kernel's algorithmic bytes (HBM-bound kernels) or FP64 instructions
(FP64-bound kernels). Cold-cache, serialised launches — a conservative
per-kernel figure (the step itself overlaps the hydro branch with the FMM).

usage: python scripts/star_kernel_table.py gpurun_out/star_launches.csv > profiles/r01_star_kernels.txt
"""

import csv
import json
import os
import statistics
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (algorithmic work constants)

L = 5
N = 8 << L                    # leaf lattice edge (256)
CELLS = N ** 3
SUB = CELLS // 512


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
    h = rows[0]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    t = defaultdict(list)
    for r in rows[1:]:
        name = r[ki].split("(")[0].split("::")[-1]
        if not name.startswith("k_star_stage"):
            name = name.split("<")[0]
        t[(name, r[gi])].append(
            float(r[vi].replace(",", "")) * 1e-9)

    hbm = float(bench.measured_peaks()[0].get("hbm_gbs", bench.FALLBACK_HBM_GBS)) * 1e9
    f64, _ = bench.fp64_peak()
    m2l, leaf = bench.fmm_interactions(L)
    p4, p3 = (N // 2) ** 3, (N // 4) ** 3          # level-4 / level-3 cells
    rec_raw, rec_red = 20 * 8, 18 * 8
    table = [
        # name, grid, per-step launches, bound, algorithmic work per launch, unit
        ("k_fmm_m2l", "(4688, 1, 1)", 2, "fp64", m2l * bench.M2L_FMA, "FMA"),
        ("k_fmm_leaf_mma", "(32768, 1, 1)", 2, "fp64", leaf * bench.LEAF_FMA, "FMA"),
        ("k_hydro_flux", "(296, 1, 1)", 2, "fp64", SUB * bench.HYDRO_FP64_PER_SUBGRID, "instr"),
        ("k_star_stage<1>", "(1184, 1, 1)", 1, "hbm", CELLS * 144, "B"),
        ("k_star_stage<2>", "(1184, 1, 1)", 1, "hbm", CELLS * 184, "B"),
        ("k_star_pad", "(1184, 1, 1)", 2, "hbm", 5 * 8 * (N ** 3 + (N + 4) ** 3), "B"),
        ("k_fmm_up", "(8192, 1, 1)", 2, "hbm", CELLS * 8 + p4 * (rec_raw + rec_red), "B"),
        ("k_fmm_up", "(1024, 1, 1)", 2, "hbm", p4 * rec_raw + p3 * (rec_raw + rec_red), "B"),
        ("k_fmm_down", "(8192, 1, 1)", 2, "hbm", p3 * rec_raw + 2 * p4 * rec_raw, "B"),
        ("k_fmm_down", "(1024, 1, 1)", 2, "hbm", (p3 // 8) * rec_raw + 2 * p3 * rec_raw, "B"),
    ]
    out = []
    total = 0.0
    for name, grid, per, bound, work, unit in table:
        key = next(k for k in t if k[0] == name and k[1] == grid)
        s = statistics.median(t[key])
        rate = work / s
        peak = hbm if bound == "hbm" else f64
        total += per * s
        out.append({"kernel": name, "grid": grid, "launches_per_step": per,
                    "ms": round(s * 1e3, 4), "bound": bound,
                    "algorithmic_per_launch": work, "unit": unit,
                    "achieved": rate, "peak": peak, "frac": round(rate / peak, 3)})
    print(f"# star step max_level {L} ({CELLS} cells): per-kernel rooflines from the ncu "
          f"launch list (median launch, cold cache, serialised); HBM peak {hbm / 1e9:.1f} GB/s "
          f"(MEASURED_PEAKS.json), FP64 peak {f64 / 1e12:.2f} T instr/s (tb_fp64_probe)")
    print(f"# {'kernel':<16} {'grid':<14} {'ms':>8} {'bound':>5} {'frac':>6}")
    for r in out:
        print(f"# {r['kernel']:<16} {r['grid']:<14} {r['ms']:>8.4f} {r['bound']:>5} "
              f"{r['frac']:>6.3f}")
    print(f"# listed kernels: {total * 1e3:.2f} ms per step serialised")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
