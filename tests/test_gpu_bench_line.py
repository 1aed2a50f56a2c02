"""bench.py's own arm on the B200 (the driver's contract): one JSON line with
the metric / unit / value / roofline / cpu_baseline / e2e / gpu_launches /
clocks keys, parity gate true, the timed region's clock record non-empty, and
the workload's numbers consistent with each other. A short run (no
ablations, no north_star kernel lines)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5",
                          "--warmup", "3", "--no-ablation", "--no-kernels"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    import bench
    assert d["metric"] == bench.METRIC and d["unit"] == "cells/s"
    assert d["higher_is_better"] is True and d["n_gpus"] == 1 and d["steps"] == 5
    assert d["dtype"] == "f64" and d["vs_baseline"] is None
    cells = d["config"]["cells"]
    assert cells == d["config"]["subgrids"] * 512
    # value = cells per second of the timed steps
    assert abs(d["value"] - cells / (d["ms_per_step"] * 1e-3)) <= 1e-6 * d["value"]
    assert d["parity"]["run_reference_512x15_equals_GOLDEN_DEFAULTS"] is True
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.05
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == cells * 8
    assert e["d2h_bytes_per_step"] >= cells * 8
    assert d["gpu_launches"] >= d["steps"]
    c = d["clocks"]
    assert c["samples"] > 0 and c["sm_mhz"] and c["sm_max_mhz"]
