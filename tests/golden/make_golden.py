"""Generate tests/golden/*.json|npz by importing the REFERENCE itself.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):  ``python tests/golden/make_golden.py``. The outputs are committed;
nothing at test/bench time reads ``/root/reference``.

What is captured (all floats as ``float.hex``):

* the reference tests' own golden literals (pkg/tests/test_miniapp.py:21-25)
  re-derived from ``taskbridge.reference.run_reference``;
* ``run_reference`` at the BASELINE configs restated as sub-grid counts
  (S = 8^L for max_level L) — C1 512x1, C2 4096x1,
  C4 32768x1, C5 262144x1 — plus 1x2, 3x3, 64x3;
* per-cell final state and per-sub-grid (min, sum) of the reference MACHINE
  (``run_scenario`` on the virtual device, src/miniapp.py:185-229) for small
  cases, read from ``Scenario.grids[i].cells`` (src/miniapp.py:132);
* per-value aggregation results of ``AggregationExecutor`` (the
  ``test_executors.py:133-147`` scenario) and the machine's per-step
  launch/transfer counts (test_miniapp.py:65-75, test_acceptance.py:43-56).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

from taskbridge.cli import RunConfig, run_single                 # noqa: E402
from taskbridge.device import ClockMode                          # noqa: E402
from taskbridge.miniapp import KERNEL_C1, KERNEL_C2              # noqa: E402
from taskbridge.reference import run_reference                   # noqa: E402
from taskbridge import (                                         # noqa: E402
    AggregationExecutor, BufferPool, ExecutorPool, Integration,
    IntegrationMode, Runtime, VirtualClockPump, VirtualDevice, build_scenario,
    ScenarioConfig, kernel_transform, run_scenario, make_kernel, when_all)


def hx(x: float) -> str:
    return float(x).hex()


def reference_runs():
    out = {}
    cases = [(1, 2), (3, 3), (4, 2), (8, 2), (64, 3), (512, 1), (512, 15),
             (4096, 1), (32768, 1), (262144, 1)]
    for s, n in cases:
        t0 = time.perf_counter()
        cs, dts = run_reference(s, n)
        wall = time.perf_counter() - t0
        out[f"{s}x{n}"] = {"subgrids": s, "steps": n, "checksum": hx(cs),
                           "dts": [hx(d) for d in dts],
                           "ref_wall_s": round(wall, 4)}
        print(f"run_reference({s},{n}) = {hx(cs)}  {wall:.2f}s", flush=True)
    return out


def machine_run(subgrids, steps, workers=2, executors=2, max_agg=4,
                mode=IntegrationMode.POLLING):
    runtime = Runtime(workers, seed=7)
    device = VirtualDevice(clock_mode=ClockMode.VIRTUAL)
    try:
        integ = Integration(runtime, device, mode)
        pool = ExecutorPool(integ, executors)
        bufs = BufferPool(device)
        aggs = [AggregationExecutor(ex, max_agg, bufs) for ex in pool.executors]
        for a in aggs:
            for k in range(5):
                a.register_kind(k, kernel_transform(k))
        sc = build_scenario(ScenarioConfig(subgrids=subgrids, steps=steps))
        by_grid = [aggs[i % len(aggs)] for i in range(subgrids)]
        pump = VirtualClockPump(runtime, device, watchdog_seconds=120.0)
        res = run_scenario(sc, runtime, device, aggs, by_grid, pump)
        cells = np.stack([g.cells for g in sc.grids])
        return res, cells
    finally:
        runtime.shutdown()
        device.destroy()


def per_subgrid_stats(subgrids):
    """One step of the reference data path at S sub-grids, per-sub-grid min/sum
    (the values _subgrid_body returns, src/miniapp.py:133)."""
    scale = float(subgrids * 1000 + 512)
    grids = [(i * 1000.0 + np.arange(512, dtype=np.float64)) / scale
             for i in range(subgrids)]
    faces = [(g[:8].copy(), g[-8:].copy()) for g in grids]
    mins, sums = [], []
    for i, g in enumerate(grids):
        work = g.copy()
        work[:8] = 0.5 * (work[:8] + faces[(i - 1) % subgrids][1])
        work[-8:] = 0.5 * (work[-8:] + faces[(i + 1) % subgrids][0])
        for _c in range(3):
            for k in range(5):
                work *= KERNEL_C1[k]
                work += KERNEL_C2[k]
        mins.append(hx(float(work.min())))
        sums.append(hx(float(work.sum())))
    return mins, sums


def aggregation_values():
    """test_executors.py:133-147 scenario: 17 requests, M=8, kind 0."""
    runtime = Runtime(2, seed=7)
    device = VirtualDevice(clock_mode=ClockMode.VIRTUAL)
    try:
        integ = Integration(runtime, device, IntegrationMode.POLLING)
        pool = ExecutorPool(integ, 1)
        agg = AggregationExecutor(pool.executors[0], 8, BufferPool(device))
        for k in range(5):
            agg.register_kind(k, kernel_transform(k))
        agg.executor.one_way(make_kernel(100_000))
        srcs = [np.full(4, float(i)) for i in range(17)]
        dsts = [np.empty(4) for _ in range(17)]
        futs = [agg.schedule(0, srcs[i], dsts[i]) for i in range(17)]
        VirtualClockPump(runtime, device).drive(when_all(futs, pool=runtime.pool))
        return {"batch_sizes_sorted": sorted(agg.batch_sizes),
                "reasons": dict(agg.reasons),
                "dst": [[hx(v) for v in d] for d in dsts]}
    finally:
        runtime.shutdown()
        device.destroy()


def counts_512():
    """criterion 1 (test_acceptance.py:43-56): unfused counts at S=512."""
    res = run_single(RunConfig(workers=8, executors=32, max_agg=1, subgrids=512,
                               steps=1, clock=ClockMode.VIRTUAL))
    m = res.per_step[0]
    return {"kernels": m.launches, "transfers": m.transfers,
            "checksum": hx(res.checksum)}


def main():
    golden = {
        "source": "generated by tests/golden/make_golden.py from /root/reference "
                  "(taskbridge 0.1.0, numpy %s)" % np.__version__,
        "reference_test_literals": {
            # pkg/tests/test_miniapp.py:21-25
            "GOLDEN_4X2": "0x1.8e6968eb86d56p+10",
            "GOLDEN_4X2_DTS": ["0x1.d0d57314f3d28p-10", "0x1.d0df8d332e761p-10"],
            "GOLDEN_8X2": "0x1.c3ca375ee34d4p+11",
            "GOLDEN_DEFAULTS": "0x1.df1096d8fa699p+20",
        },
        "run_reference": reference_runs(),
    }
    mins, sums = per_subgrid_stats(64)
    golden["per_subgrid_64x1"] = {"mins": mins, "sums": sums}
    golden["aggregation_17_m8"] = aggregation_values()
    golden["machine_counts_512x1_m1"] = counts_512()

    machine = {}
    arrays = {}
    for (s, n, w, e, m) in [(4, 2, 2, 2, 8), (8, 2, 2, 1, 4), (1, 2, 1, 1, 2),
                            (16, 3, 4, 4, 4)]:
        res, cells = machine_run(s, n, workers=w, executors=e, max_agg=m)
        key = f"{s}x{n}"
        machine[key] = {
            "checksum": hx(res.checksum), "dts": [hx(d) for d in res.dts],
            "launches": [p.launches for p in res.per_step],
            "transfers": [p.transfers for p in res.per_step],
            "workers": w, "executors": e, "max_agg": m}
        arrays[f"cells_{key}"] = cells
        print(f"machine {key}: {hx(res.checksum)}", flush=True)
    golden["machine"] = machine
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(golden, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "cells.npz"), **arrays)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
