#!/usr/bin/env python
"""Benchmark: sub-grid cells processed per second (FP64 ring step) on 1..N B200.

Workload (default, ``--workload c4``): BASELINE.json config 4 restated on the
pinned path: the full mini-app time step — ghost fold, 3x5
kernel chain, per-sub-grid min + numpy-order pairwise sum, exact fsum
checksum and min-tree dt — over 8^5 = 32768 sub-grids (16.8 M cells) PER GPU
on a 1-D ring partitioned contiguously across ranks (weak scaling; halo
faces by NCCL P2P, accumulator by NCCL all-reduce). ``--workload c2`` is the
4096-sub-grid batch of config 2, ``c5`` the 8^6 ring (per GPU).

One JSON line on rank 0. ``value`` = cells of all ranks per second over the
timed steps, device-timed with CUDA events (max over ranks), inputs resident
in HBM, steps back to back (each step's input, the previous step's 128 MiB
output, exceeds the 126 MB L2 and is read from DRAM in full:
profiles/r01_k2_back_to_back.txt); ``l2_flushed_per_step`` repeats the
measurement with a 256 MiB L2-flushing write before every step. ``e2e`` = the
same metric through the host-buffer API (RingStepper.step_host: pinned H2D
of the cells, step, D2H of the new cells and (piece, dt)). ``roofline`` is
the fused step kernel K2 against measured HBM bandwidth. ``cpu_baseline`` is
the C port of the reference data path (oracle/tb_oracle.c, OpenMP, all host
threads) on a bounded sample.

``--impl reference``: rank 0 times that CPU implementation on this arm's
config and prints the same line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c2": (4096, "C2: 4096 sub-grids of 8^3 cells + ring ghost faces, one full step "
                 "(ghost fold + 15 FP64 kernels + min/pairwise-sum + exact checksum)"),
    "c4": (32768, "C4: full step at max_level 5 (8^5 = 32768 sub-grids of 8^3 cells) "
                  "per GPU: ghost fold + 15 FP64 kernels + min/pairwise-sum + exact "
                  "fsum checksum + min-tree dt"),
    "c5": (262144, "C5: full step at max_level 6 (8^6 = 262144 sub-grids) per GPU"),
}
METRIC = "sub-grid cells processed/sec (rotating star, FP64) at 1/2/4/8 B200 vs CPU ref"
BYTES_PER_CELL = 8 + 8 + 0.25 + 0.03125   # 16.28 B/cell-step
# FP64 instructions per cell-step: 15 x (DMUL + DADD), the
# ghost fold (2 ops on 16 of 512 cells), one DADD of the pairwise sum, one min
FP64_PER_CELL = 30 + 2 * 16 / 512 + 2
GOLDEN_DEFAULTS = float.fromhex("0x1.df1096d8fa699p+20")   # run_reference(512, 15)
FALLBACK_HBM_GBS = 6650.0
AUTO_IMPL = "bulk1"
SCENARIO_STEPS = 15    # run_scenario's default step count (src/cli.py, GOLDEN_DEFAULTS)    # what TB_STEP_AUTO launches for the aligned (3, 5) chain


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return json.load(fh), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": FALLBACK_HBM_GBS}, "fallback"


class ClockSampler:
    """SM clock + throttle reasons around and DURING the timed region.

    NVML (``pynvml``) from a background thread every ~1 ms from before the
    warm-up to after the timed region, each sample time-stamped, plus
    samples taken on the launching thread while the timed launches are still
    executing (the host returns from the asynchronous launches long before
    the GPU finishes them, so those samples are genuinely under load) and
    one synchronous sample right before and right after. Falls back to
    ``nvidia-smi -lms 50``."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []          # (t, sm_mhz, mem_mhz, reasons bitmask)
        self._stop = None
        self._thread = None
        self._nvml = None
        self._proc = None
        self.window = None         # (t0, t1) of the timed region
        self.during = []           # samples taken while the timed launches ran
        self.edges = {}            # "before"/"after" synchronous samples

    def _read(self):
        pynvml, h = self._nvml
        return (time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))

    def sample(self, into=None):
        """One synchronous sample (appended to ``into`` or returned)."""
        if self._nvml is None:
            return None
        try:
            s = self._read()
        except Exception:  # noqa: BLE001
            return None
        if into is not None:
            into.append(s)
        return s

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self._nvml = (pynvml, h)
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - no NVML: use nvidia-smi
            self._nvml = None
        if self._nvml is None:
            try:
                q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                     "clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
                self._proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                     "--format=csv,noheader,nounits", "-lms", "50"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except OSError:
                self._proc = None
            return
        self._stop = threading.Event()

        def loop():
            while not self._stop.is_set():
                self.sample(self.samples)
                self._stop.wait(0.001)

        self._thread = threading.Thread(target=loop, daemon=True)
        self._thread.start()

    def _names(self, rows):
        pynvml = self._nvml[0]
        return sorted({name for *_, rs in rows for name, attr in self.REASONS.items()
                       if rs & getattr(pynvml, attr, 0)})

    def stop(self):
        if self._nvml is not None:
            self._stop.set()
            self._thread.join(timeout=2)
            t0, t1 = self.window if self.window else (float("-inf"), float("inf"))
            inside = [s for s in self.samples if t0 <= s[0] <= t1] + self.during
            near = [s for s in self.samples if t0 - 0.05 <= s[0] <= t1 + 0.05]
            use = inside or near
            sm = [s[1] for s in use]
            return {"sm_mhz": statistics.median(sm) if sm else None,
                    "sm_max_mhz": self._max,
                    "mem_mhz": statistics.median(s[2] for s in use) if use else None,
                    "reasons": self._names(use + list(self.edges.values())),
                    "samples": len(inside), "samples_within_50ms": len(near),
                    "before": self.edges.get("before", (None, None))[1],
                    "after": self.edges.get("after", (None, None))[1],
                    "source": "nvml: 1 ms thread + launching-thread samples while the "
                              "timed launches run + before/after"}
        if self._proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock source"],
                    "samples": 0}
        self._proc.terminate()
        try:
            out, _ = self._proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self._proc.kill()
            out, _ = self._proc.communicate()
        rows = [[p.strip() for p in ln.split(",")] for ln in out.strip().splitlines()]
        rows = [r for r in rows if len(r) >= 6]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max((float(r[1]) for r in rows
                                   if r[1].replace(".", "").isdigit()), default=None),
                "reasons": sorted({names[i] for r in rows for i in range(4)
                                   if r[2 + i].lower() == "active"}),
                "samples": len(rows), "source": "nvidia-smi/50ms"}


def cpu_reference_sample(subgrids: int, budget_s: float, threads: int = 0):
    """Time the C port of the reference data path (oracle/tb_oracle.c) on the
    host: repeated full steps of ``subgrids`` sub-grids until ``budget_s``."""
    import numpy as np
    from oracle import c_oracle
    threads = threads or len(os.sched_getaffinity(0))
    old = c_oracle.init_cells(subgrids)
    new = np.empty_like(old)
    mins, sums = np.empty(subgrids), np.empty(subgrids)
    steps, t0 = 0, time.perf_counter()
    while True:
        c_oracle.step(old, new, old[-1, -8:].copy(), old[0, :8].copy(), mins, sums,
                      threads=threads)
        c_oracle.fsum(sums)
        old, new = new, old
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return subgrids * 512 * steps / el, threads, steps, el


def python_reference_sample(subgrids: int = 4096, budget_s: float = 3.0):
    """The north_star's "Python CPU reference timed on the box's own host
    cores": src/reference.py:23-50 restated with its execution shape (a
    Python loop of 512-value numpy ops per sub-grid,
    oracle/miniapp_oracle.run_reference_per_subgrid, equal to the pinned
    oracle; the reference package itself cannot travel to the GPU box). One
    core: numpy runs these ops single-threaded. Repeated one-step runs of
    ``subgrids`` sub-grids until ``budget_s``."""
    from oracle import miniapp_oracle as mo
    runs, t0 = 0, time.perf_counter()
    while True:
        mo.run_reference_per_subgrid(subgrids, 1)
        runs += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return {"value": subgrids * 512 * runs / el, "unit": "cells/s", "cores": 1,
            "kind": "port (src/reference.py:23-50 restated, per-sub-grid numpy loop)",
            "sample": f"{runs} x run_reference({subgrids}, 1) in {el:.1f}s "
                      "(initialisation included, as in the reference)"}


def machine_ablation(subgrids=512, steps=6, repeats=5, workers=(2, 4, 8)):
    """The paper's ablation in the same run: the mini-app machine (native C++
    runtime, tb_machine_run) at the paper's scenario size (512 sub-grids,
    PAPER.md:775-782) with the paper's best combination, 32 executors x max 8
    aggregated, completion by POLLING vs HOSTTASK vs FENCE — at 8 workers
    (the top-level keys) and, as the paper's third graph does (PAPER.md:
    931-941), with fewer workers, where a fence-blocked worker weighs more.
    Median of `repeats` runs of the mean step time over steps 2..N."""
    from paper_2303_08058_b200.bridge import IntegrationMode
    from paper_2303_08058_b200.native_machine import run_native
    out = {"config": f"native machine, {subgrids} sub-grids x {steps} steps, 32 executors, "
                     f"max 8 aggregated, staged batches, workers {list(workers)}, median of "
                     f"{repeats}"}
    checks = set()

    def cell(W, mode, zero_copy=0, completion="events"):
        ms = []
        for _ in range(repeats):
            res, _ = run_native(subgrids, steps, workers=W, executors=32, max_agg=8,
                                mode=mode, zero_copy=zero_copy, completion=completion)
            ms.append(statistics.fmean(res.step_ms[1:]))
            checks.add(res.checksum.hex())
        return statistics.median(ms)

    sweep = {}
    for W in workers:
        row = {f"{m.value}_ms_per_step": cell(W, m) for m in
               (IntegrationMode.POLLING, IntegrationMode.HOSTTASK, IntegrationMode.FENCE)}
        row["speedup_polling_vs_fence"] = row["fence_ms_per_step"] / row["polling_ms_per_step"]
        row["speedup_hosttask_vs_fence"] = row["fence_ms_per_step"] / row["hosttask_ms_per_step"]
        sweep[f"W{W}"] = row
    out.update(sweep[f"W{max(workers)}"])
    out["workers_sweep"] = sweep
    # the same machine with zero-copy batches at 8 workers: each batch kernel
    # in place on its pinned staging buffer (one launch + one event per batch
    # instead of H2D ; kernel ; D2H)
    zc = {f"{m.value}_ms_per_step": cell(max(workers), m, 1)
          for m in (IntegrationMode.POLLING, IntegrationMode.FENCE)}
    zc["speedup_polling_vs_fence"] = zc["fence_ms_per_step"] / zc["polling_ms_per_step"]
    out["zero_copy"] = zc
    # the B200 machine's own batches on the same scenario and sweep: direct
    # (no host copies of the cells) with completion by CUDA events and by
    # kernel-stored completion words (no event records or queries)
    direct = {}
    for W in workers:
        row = {}
        for comp in ("events", "words"):
            for m in (IntegrationMode.POLLING, IntegrationMode.FENCE):
                row[f"{comp}_{m.value}_ms_per_step"] = cell(W, m, 4, comp)
            row[f"{comp}_speedup_polling_vs_fence"] = (row[f"{comp}_fence_ms_per_step"]
                                                       / row[f"{comp}_polling_ms_per_step"])
        direct[f"W{W}"] = row
    out["direct"] = direct
    out["checksums_identical"] = len(checks) == 1
    return out


# BASELINE config 4 (max_level 5) on the native machine with the reference
# task structure; run_reference(32768, 1) pins step 1
C4_CHECKSUM = float.fromhex("0x1.fffc131fd56c6p+22")
C4_DT = float.fromhex("0x1.a73380416f1a6p-22")
# the sweeps' best polling configuration (scripts/c4_machine_sweep.py,
# c4_gather_sweep.py, c4_resident_sweep.py, c4_direct_probe.py;
# profiles/r02/c4_*): 8 workers — half the box's 16 host cores: the machine
# saturates there (15.2 ms/step vs 14.8 at 16 workers), and, as in the
# paper's best-combination test, the other half is what a fence-blocked
# worker would otherwise leave the host (16 workers are in the sweep) —
# 8 executors, max 512 aggregated (two gather launches of 256 per batch;
# 12.4 ms/step against 14.8 at 256 and 11.9 at 1024, where polling and
# fence draw level: profiles/r02/c4_m_probe.txt, c4_m_ablation_probe.txt),
# direct batches (each task's rounds between the first and the last stay in
# HBM; the first round's kernel reads the pinned rows and folds the ghost
# faces, the last writes them back with min and pairwise sum — no host copy
# of the cells; gather batches move every round over PCIe: 4 GB per step, a
# 40 ms floor; resident = direct with the fold / reductions on the host)
C4_MACHINE = dict(workers=8, executors=8, max_agg=512, zero_copy=4)
C4_SWEEP = [(4, 8), (16, 8), (16, 16)]   # (workers, executors) beside C4_MACHINE


def machine_ablation_c4(steps=4, repeats=3):
    """The paper's ablation at BASELINE config 4: the native machine on 32768
    sub-grids with the reference task structure (one task and 15 schedule()
    calls per sub-grid per step, src/miniapp.py:116-171, driven as
    src/cli.py:199-232), POLLING vs HOSTTASK vs FENCE at identical
    (W, E, M), completion by CUDA events (the paper's mechanism) and by
    kernel-stored completion words (words_*); gather batches (every round over PCIe) under POLLING and FENCE
    and the staged op sequence (H2D ; kernel ; D2H per batch) under POLLING at
    the same (W, E, M); and a (workers, executors) sweep. A run's time is the
    mean step time over steps 2..N; each cell is the median of `repeats`
    runs, the runs of the modes compared interleaved (a host-side scheduler
    on a shared box is noisy: one run to the next varies by up to 1.5x,
    profiles/r02/c4_context_probe.txt). Speed-ups = fence_ms / mode_ms
    (src/cli.py:297-306); parity: every run's first step equals
    run_reference(32768, 1)."""
    from paper_2303_08058_b200.bridge import IntegrationMode
    from paper_2303_08058_b200.native_machine import run_native
    P, H, F = IntegrationMode.POLLING, IntegrationMode.HOSTTASK, IntegrationMode.FENCE
    out = {"config": "native machine, 32768 sub-grids (max_level 5), reference task structure "
                     f"(491,520 schedule() calls per step), {C4_MACHINE['workers']} workers, "
                     f"{C4_MACHINE['executors']} executors, max {C4_MACHINE['max_agg']} "
                     "aggregated, direct batches (rounds 2..14 of each task in HBM; round 1 reads "
                     "the pinned rows and folds the ghost faces in its kernel, round 15 writes "
                     "them back with min and pairwise sum), "
                     f"{steps} steps (mean of steps 2..{steps}), "
                     f"median of {repeats} interleaved runs"}
    checks, golden = set(), [True]

    def compare(cells):
        """cells: [(name, mode, machine kwargs)] -> {name: (median ms, last run)}"""
        ms = {name: [] for name, _, _ in cells}
        last = {}
        for _ in range(repeats):
            for name, mode, kw in cells:
                res, _ = run_native(32768, steps, mode=mode, **kw)
                ms[name].append(statistics.fmean(res.step_ms[1:]))
                last[name] = res
                checks.add(res.checksum.hex())
                golden[0] &= (res.per_step[0].checksum_piece == C4_CHECKSUM
                              and res.dts[0] == C4_DT)
        return {name: (statistics.median(v), last[name]) for name, v in ms.items()}

    main = compare([(m.value, m, C4_MACHINE) for m in (P, H, F)]
                   + [("words_polling", P, dict(C4_MACHINE, completion="words")),
                      ("words_fence", F, dict(C4_MACHINE, completion="words")),
                      ("resident_polling", P, dict(C4_MACHINE, zero_copy=3)),
                      ("resident_fence", F, dict(C4_MACHINE, zero_copy=3)),
                      ("gather_polling", P, dict(C4_MACHINE, zero_copy=2)),
                      ("gather_fence", F, dict(C4_MACHINE, zero_copy=2))])
    main.update(compare([("staged_polling", P, dict(C4_MACHINE, zero_copy=0))]))
    for name, (ms, res) in main.items():
        out[f"{name}_ms_per_step"] = ms
        out[f"{name}_mean_batch"] = res.per_step[-1].mean_batch
        out[f"{name}_launches_per_step"] = res.per_step[-1].launches
    out["speedup_polling_vs_fence"] = out["fence_ms_per_step"] / out["polling_ms_per_step"]
    out["speedup_hosttask_vs_fence"] = out["fence_ms_per_step"] / out["hosttask_ms_per_step"]
    out["words_speedup_polling_vs_fence"] = (out["words_fence_ms_per_step"]
                                             / out["words_polling_ms_per_step"])
    out["resident_speedup_polling_vs_fence"] = (out["resident_fence_ms_per_step"]
                                                / out["resident_polling_ms_per_step"])
    out["gather_speedup_polling_vs_fence"] = (out["gather_fence_ms_per_step"]
                                              / out["gather_polling_ms_per_step"])
    out["cells_per_s_polling"] = 32768 * 512 / (out["polling_ms_per_step"] * 1e-3)
    # the same at other (workers, executors): where a fence-blocked worker
    # weighs more or less (polling and fence at identical settings)
    sweep = {}
    for W, E in C4_SWEEP:
        kw = dict(C4_MACHINE, workers=W, executors=E)
        kww = dict(kw, completion="words")
        r = compare([("polling", P, kw), ("fence", F, kw), ("words_polling", P, kww),
                     ("words_fence", F, kww)])
        row = {k + "_ms_per_step": v[0] for k, v in r.items()}
        row["speedup_polling_vs_fence"] = row["fence_ms_per_step"] / row["polling_ms_per_step"]
        row["words_speedup_polling_vs_fence"] = (row["words_fence_ms_per_step"]
                                                 / row["words_polling_ms_per_step"])
        sweep[f"W{W}_E{E}"] = row
    out["sweep"] = sweep
    out["checksums_identical"] = len(checks) == 1
    out["step1_equals_run_reference_32768x1"] = golden[0]
    return out


PCIE_BIDIR_GBS = 99.86   # measured concurrent H2D + D2H (profiles/r01/pcie_probe.json)


def plugin_call_bench(steps=3):
    """e2e through the reference's own plugin/operator API at BASELINE config
    4: build_scenario + Runtime + CudaDevice + Integration(POLLING) +
    ExecutorPool + AggregationExecutor(register_kind(k, kernel_transform(k)))
    + run_scenario, wired as src/cli.py:199-232 does, on 32768 sub-grids
    whose cells live in host memory (the reference's Scenario.grids). The
    call delegates to the native machine (miniapp._native_plan). "staged"
    and "gather": every kernel round moves each sub-grid's 4 KiB over PCIe
    and back, 15 rounds per step (the reference's op sequence) — the bound
    stated below; "resident": the task's rounds between the first and the
    last stay in HBM (two PCIe crossings per sub-grid and step); "direct":
    resident with the ghost fold and the per-sub-grid min / pairwise sum in
    the first / last round's kernel, on the Scenario's pinned rows (no host
    copy of the cells). The build_scenario call (which pins the rows) is
    outside the timed call, as the reference's scenario construction is."""
    from paper_2303_08058_b200 import (AggregationExecutor, BufferPool, CudaDevice,
                                       ExecutorPool, Integration, IntegrationMode, Runtime,
                                       ScenarioConfig, build_scenario, kernel_transform,
                                       run_scenario)
    S = 32768
    W, E, M = C4_MACHINE["workers"], C4_MACHINE["executors"], C4_MACHINE["max_agg"]
    out = {"api": "run_scenario(build_scenario(ScenarioConfig(subgrids=32768, steps="
                  f"{steps})), Runtime({W}), CudaDevice(0), aggs=[AggregationExecutor(ex, {M}, "
                  f"BufferPool) for ex in ExecutorPool(Integration(POLLING), {E})], "
                  "round-robin aggs_by_grid) -> native machine (reference task structure)",
           "unit": "cells/s"}
    pcie_bytes = S * 15 * 512 * 8 * 2
    for copies, completion in (("direct", "events"), ("direct", "words"), ("resident", "events"),
                               ("gather", "events"), ("staged", "events"), ("fused", "events")):
        rt = Runtime(W)
        dev = CudaDevice(0)
        try:
            integ = Integration(rt, dev, IntegrationMode.POLLING)
            pool = ExecutorPool(integ, E)
            bufs = BufferPool(dev)
            aggs = [AggregationExecutor(ex, M, bufs) for ex in pool.executors]
            for a in aggs:
                for k in range(5):
                    a.register_kind(k, kernel_transform(k))
            sc = build_scenario(ScenarioConfig(subgrids=S, steps=steps))
            t0 = time.perf_counter()
            if copies == "fused":     # the aggregation machine bypassed: one K2 per step
                res = run_scenario(sc, rt, dev, aggs, [aggs[g % E] for g in range(S)],
                                   engine="fused")
            else:
                res = run_scenario(sc, rt, dev, aggs, [aggs[g % E] for g in range(S)],
                                   batch_copies=copies, completion=completion)
            call_s = time.perf_counter() - t0
        finally:
            rt.shutdown()
            dev.destroy()
        step_ms = statistics.fmean(res.step_ms[1:])
        key = copies if completion == "events" else f"{copies}_{completion}"
        out[key] = {"ms_per_step": step_ms, "value": S * 512 / (step_ms * 1e-3),
                       "completion": completion,
                       "call_s": call_s, "call_value": S * 512 * steps / call_s,
                       "engine": res.engine, "batch_copies": res.batch_copies,
                       "step1_equals_run_reference_32768x1":
                           res.per_step[0].checksum_piece == C4_CHECKSUM
                           and res.dts[0] == C4_DT}
    # the call's value: the fastest bit-identical variant through run_scenario
    best = max(("direct", "direct_words", "resident"), key=lambda k: out[k]["value"])
    out["value"] = out[best]["value"]
    out["value_mode"] = best
    out["h2d_bytes_per_step"] = S * 512 * 8
    out["d2h_bytes_per_step"] = S * 512 * 8
    out["direct"]["pcie_bytes_per_step"] = 2 * S * 512 * 8
    out["direct_words"]["pcie_bytes_per_step"] = 2 * S * 512 * 8
    out["fused"]["pcie_bytes_per_step"] = 2 * S * 512 * 8 / steps
    out["fused"]["note"] = ("run_scenario(engine='fused'): the grids uploaded once per call, "
                            "one K2 launch of all sub-grids per step, the grids read back; "
                            "bypasses the aggregation machine (not in `value`); per-step "
                            "time = the call's device time / steps")
    out["resident"]["pcie_bytes_per_step"] = 2 * S * 512 * 8
    out["gather"]["pcie_bytes_per_step"] = pcie_bytes
    out["staged"]["pcie_bytes_per_step"] = pcie_bytes
    out["bound"] = {"kind": "pcie", "bytes_per_step": pcie_bytes,
                    "measured_bidirectional_gbs": PCIE_BIDIR_GBS,
                    "floor_ms": pcie_bytes / (PCIE_BIDIR_GBS * 1e9) * 1e3,
                    "frac": pcie_bytes / (PCIE_BIDIR_GBS * 1e9) * 1e3
                    / out["gather"]["ms_per_step"],
                    "applies_to": "gather and staged",
                    "why": "15 kernel rounds per sub-grid per step, each a host->device->host "
                           "trip of its 4 KiB (the reference machine's structure, "
                           "src/miniapp.py:127-131, src/executors.py:257-284)"}
    return out


HYDRO_BYTES_PER_SUBGRID = 5 * 12 ** 3 * 8 + 5 * 8 ** 3 * 8 + 8   # U in, dU/dt + amax out

def hydro_fp64_per_subgrid():
    """FP64 instructions per sub-grid of the K6 spec (oracle/hydro_oracle.py),
    an IEEE divide / square root counted as the 8-instruction sequence it
    executes (tb_internal.h div_rn_fast / sqrt_rn_fast); the minmod compares
    (2 per slope) and the signal-speed maxima (2 per face) counted too — they
    issue on the FP64 pipe. DESIGN.md K6."""
    cells, faces = 12 ** 3, 3 * 9 * 8 * 8
    convert = 8 + 3 + 6 + 2                 # 1/rho, v = s/rho, ke, p
    state = 1 + 8 + 8 + 5 + 4 + 3 + 4 + 1 + 2 + 1   # cs, |v|^2, e, m, momentum/energy flux, a
    flux = 2 * state + 1 + 5 * 5            # two states, a/2, 5 x LLF combine
    # minmod PLM: per line segment of N faces, N+1 slopes (2 DADD + DMUL) and
    # 4 ops per face, per field; 192 segments of 2 and 64 of 3 per direction
    recon = 3 * 5 * (192 * (3 * 3 + 2 * 4) + 64 * (4 * 3 + 3 * 4))
    fold = 512 * 5 * (1 + 2 + 2) + 512 * 5  # flux differences + the 1/dx scaling
    compares = 3 * 5 * (192 * 3 + 64 * 4) * 2 + faces * 2
    return cells * convert + faces * flux + recon + fold + compares


HYDRO_FP64_PER_SUBGRID = hydro_fp64_per_subgrid()
# the same spec counted as operations: each IEEE divide / square root is ONE
# op instead of its 8-instruction sequence — 1,728 reciprocals (1/rho per
# staged cell) + 3 x 576 faces x 2 states x (one divide + one square root)
HYDRO_DIVSQRT_PER_SUBGRID = 12 ** 3 + 3 * 576 * 2 * 2
HYDRO_FP64_OPS_PER_SUBGRID = HYDRO_FP64_PER_SUBGRID - 7 * HYDRO_DIVSQRT_PER_SUBGRID
M2L_FMA, LEAF_FMA = 70, 4     # algorithmic FP64 FMAs per interaction (traceless M2L, K7)


def fp64_peak():
    """Measured FP64 issue rate (profiles/fp64_peak.json, tb_fp64_probe)."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as fh:
            return json.load(fh)["dfma_instr_per_s"], "measured (tb_fp64_probe)"
    except (OSError, ValueError, KeyError):
        return 64 * 148 * 1.965e9, "nominal 64 DFMA/clk/SM x 148 SMs x 1965 MHz"


def fmm_interactions(L):
    """Algorithmic interaction counts of the FMM at max_level L: (M2L pairs of
    levels 0..L-1 on the interaction lists, leaf monopole pairs)."""
    import itertools
    pnear = [p for p in itertools.product(range(-2, 3), repeat=3) if sum(x * x for x in p) <= 4]
    ch = list(itertools.product((0, 1), repeat=3))

    def inside(v, n):
        return 0 <= v < n

    m2l = 0
    # level 0: every far pair of the 8^3 root lattice
    g = list(itertools.product(range(8), repeat=3))
    m2l += sum(1 for a in g for b in g if sum((a[k] - b[k]) ** 2 for k in range(3)) > 4)
    for lev in range(1, L):
        n = 8 << lev
        # per parent position along an axis the in-range count factorises only
        # approximately; count exactly over one axis-symmetric sweep
        tot = 0
        for o in ch:
            for P in pnear:
                for c in ch:
                    q = [o[k] - 2 * P[k] - c[k] for k in range(3)]
                    if sum(x * x for x in q) <= 4:
                        continue
                    cnt = 1
                    for k in range(3):   # targets along axis k whose partner is in range
                        cnt *= sum(1 for i in range(o[k], n, 2) if inside(i - q[k], n))
                    tot += cnt
        m2l += tot
    nl = 8 << L
    leaf = 0
    for o in ch:
        for P in pnear:
            for c in ch:
                q = [o[k] - 2 * P[k] - c[k] for k in range(3)]
                if q == [0, 0, 0]:
                    continue
                cnt = 1
                for k in range(3):
                    cnt *= sum(1 for i in range(o[k], nl, 2) if inside(i - q[k], nl))
                leaf += cnt
    return m2l, leaf


def north_star_kernels(dev, reps=20):
    """BASELINE configs 2 and 3 on the north_star's hydro (K6) and FMM (K7)
    kernels — PARITY UNPINNED (self-authored specs, oracle/hydro_oracle.py,
    oracle/fmm_oracle.py; the reference has neither). CUDA events on the
    launching stream, L2 flushed before every timed launch."""
    import torch
    from paper_2303_08058_b200 import hydro
    from paper_2303_08058_b200.gravity import GravitySolver, rotating_star_density
    peaks, _ = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
    f64, f64_src = fp64_peak()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {}
    # K6: hydro reconstruct+flux, 4096 sub-grids (config 2)
    S = 4096
    I, dx = hydro.rotating_star(S, device=dev)
    U = hydro.with_ghosts(I)
    du = torch.empty((S, 5, 8, 8, 8), dtype=torch.float64, device=dev)
    am = torch.empty(S, dtype=torch.float64, device=dev)
    for _ in range(3):
        hydro.hydro_flux(U, dx, out=du, amax=am)
    # back to back, as the K2 headline: the 283 MB input exceeds the 126 MB
    # L2 and every launch reads all of it from DRAM (ncu --cache-control
    # none: 283.1 MB read per launch, profiles/r02/k6_b2b_probe.txt); the
    # L2-flushed figure (a 256 MiB write before each launch) beside it
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        hydro.hydro_flux(U, dx, out=du, amax=am)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        hydro.hydro_flux(U, dx, out=du, amax=am)
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    ms_flushed = tot / reps
    gbs = S * HYDRO_BYTES_PER_SUBGRID / (ms * 1e-3) / 1e9
    out["hydro_k6"] = {
        "config": "BASELINE config 2: hydro reconstruct+flux, 4096 synthetic 8^3 sub-grids "
                  "with 2-cell ghost layers (rotating star), 1 B200",
        "kernel": "k_hydro_flux", "ms": ms, "cells_per_s": S * 512 / (ms * 1e-3),
        "l2": "launches back to back, input (283 MB) larger than L2: every launch reads it "
              "all from DRAM (ncu --cache-control none: 283.1 MB per launch)",
        "l2_flushed": {"ms": ms_flushed,
                       "fp64_frac": S * HYDRO_FP64_PER_SUBGRID / (ms_flushed * 1e-3) / f64,
                       "method": "256 MiB write before each launch, events per launch"},
        "roofline": {"bound": "fp64 (divide/sqrt-heavy; see profiles)", "hbm_achieved_gbs": gbs,
                     "hbm_frac": gbs / hbm,
                     "fp64_instr_per_subgrid": HYDRO_FP64_PER_SUBGRID,
                     "fp64_achieved": S * HYDRO_FP64_PER_SUBGRID / (ms * 1e-3),
                     "fp64_peak": f64, "fp64_peak_source": f64_src,
                     "fp64_frac": S * HYDRO_FP64_PER_SUBGRID / (ms * 1e-3) / f64,
                     "fp64_ops_per_subgrid": HYDRO_FP64_OPS_PER_SUBGRID,
                     "fp64_ops_frac": S * HYDRO_FP64_OPS_PER_SUBGRID / (ms * 1e-3) / f64,
                     "fp64_frac_note": "fp64_frac: issued FP64 instructions (a divide or square "
                                       "root = its 8-instruction sequence, the rate the FP64 "
                                       "pipe sees); fp64_ops_frac: spec operations (a divide "
                                       "or square root = 1 op), against the same peak",
                     "algorithmic_bytes_per_launch": S * HYDRO_BYTES_PER_SUBGRID},
        "parity": "unpinned (self-authored spec; bit-exact to oracle/hydro_oracle.py)"}
    # the same kernel at the star step's size (max_level 5, 32768 sub-grids):
    # the per-launch head (every CTA's first staging, 3-8 us) and the last
    # wave's granularity (CTAs finish up to ~1.4 sub-grids apart even with
    # dynamic assignment; profiles/r02/k6_experiments.md) are ~7 % of a
    # config-2 launch and ~1 % here
    del U, du, am
    S5 = 8 ** 5
    I5, dx5 = hydro.rotating_star(S5, device=dev)
    U5 = hydro.with_ghosts(I5)
    del I5
    du5 = torch.empty((S5, 5, 8, 8, 8), dtype=torch.float64, device=dev)
    am5 = torch.empty(S5, dtype=torch.float64, device=dev)
    hydro.hydro_flux(U5, dx5, out=du5, amax=am5)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        hydro.hydro_flux(U5, dx5, out=du5, amax=am5)
    b.record()
    torch.cuda.synchronize()
    ms5 = a.elapsed_time(b) / 5
    out["hydro_k6"]["max_level_5"] = {
        "subgrids": S5, "ms": ms5, "cells_per_s": S5 * 512 / (ms5 * 1e-3),
        "fp64_frac": S5 * HYDRO_FP64_PER_SUBGRID / (ms5 * 1e-3) / f64,
        "fp64_ops_frac": S5 * HYDRO_FP64_OPS_PER_SUBGRID / (ms5 * 1e-3) / f64,
        "note": "same kernel, launches back to back (2.26 GB input) at 32768 sub-grids "
                "(the star step's max_level-5 lattice size): the config-2 launch carries "
                "its head (first staging of every CTA) and last-wave tail, ~7 us"}
    del U5, du5, am5
    # K7: FMM gravity, max_level 4 (config 3)
    L = 4
    rho = rotating_star_density(L, device=dev)
    gs = GravitySolver(L, dev)
    for _ in range(3):
        gs.solve(rho)
    names = ["upward", "m2l", "downward", "leaf"]
    acc = dict.fromkeys(names + ["solve"], 0.0)
    for _ in range(reps):
        flush.fill_(1)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        gs.upward(rho)
        ev[1].record()
        gs.m2l()
        ev[2].record()
        gs.downward()
        ev[3].record()
        gs.leaf(rho)
        ev[4].record()
        torch.cuda.synchronize()
        for i, k in enumerate(names):
            acc[k] += ev[i].elapsed_time(ev[i + 1])
        acc["solve"] += ev[0].elapsed_time(ev[4])
    ms = {k: v / reps for k, v in acc.items()}
    nm, nl = fmm_interactions(L)
    m2l_rate = nm * M2L_FMA / (ms["m2l"] * 1e-3)
    leaf_rate = nl * LEAF_FMA / (ms["leaf"] * 1e-3)
    cells = (8 << L) ** 3
    out["fmm_k7"] = {
        "config": "BASELINE config 3: FMM multipole (M2L, levels 0-3) + monopole (leaf) "
                  "interaction kernels, rotating star max_level 4 (2,097,152 leaf cells), 1 B200",
        "ms": ms, "cells_per_s": cells / (ms["solve"] * 1e-3),
        "interactions": {"m2l": nm, "leaf": nl},
        "roofline": {"bound": "fp64", "unit": "DFMA/s", "peak": f64, "peak_source": f64_src,
                     "m2l_achieved": m2l_rate, "m2l_frac": m2l_rate / f64,
                     "leaf_achieved": leaf_rate, "leaf_frac": leaf_rate / f64,
                     "algorithmic_fma_per_interaction": {"m2l": M2L_FMA, "leaf": LEAF_FMA}},
        "gpu_launches_per_solve": 2 * L + 2,
        "parity": "unpinned (self-authored spec; 1e-10 relative to oracle/fmm_oracle.py)"}
    # the coupled rotating-star step at max_level 5 (hydro + FMM + SSP-RK2),
    # steps back to back (the 640 MiB state exceeds L2), CUDA-graph replay
    from paper_2303_08058_b200.star import RotatingStarStep
    Ls, ks = 5, 5
    st = RotatingStarStep(Ls, device=dev)
    m0 = st.U[0].sum().item()
    for _ in range(2):
        st.step(graph=True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(ks):
        st.step(graph=True)
    b.record()
    torch.cuda.synchronize()
    ms_star = a.elapsed_time(b) / ks
    m1 = st.U[0].sum().item()
    out["star_step"] = {
        "config": "north_star full rotating-star step, max_level 5 (16,777,216 cells): "
                  "periodic pad + hydro (K6, TMA boxes) + FMM gravity (K7) per SSP-RK2 stage, "
                  "on-device CFL dt, one CUDA graph per step",
        "ms_per_step": ms_star, "cells_per_s": st.n ** 3 / (ms_star * 1e-3),
        "launches_per_step": st.launches_per_step(),
        "mass_rel_drift_over_7_steps": abs(m1 - m0) / m0,
        "parity": "unpinned (self-authored spec oracle/star_oracle.py; 1e-10 per cell)"}
    del st
    return out


def hydro_machine_ablation(subgrids=512, steps=8, repeats=3):
    """The paper's experiment shape on the north_star hydro kernel (PAPER.md:
    762-782: per-sub-grid hydro tasks, aggregated launches): the native
    machine with K6 tasks (tb_machine_run_hydro; parity unpinned, bit-exact
    to oracle/hydro_oracle.py euler_step), 32 executors x max 8, 8 workers,
    POLLING vs HOSTTASK vs FENCE; median of `repeats` of the mean step time
    over steps 3..N."""
    from paper_2303_08058_b200.bridge import IntegrationMode
    from paper_2303_08058_b200.hydro import rotating_star
    from paper_2303_08058_b200.native_machine import run_native_hydro
    I = rotating_star(subgrids)[0].numpy()
    out = {"config": f"native machine, hydro (K6) tasks, {subgrids} sub-grids x {steps} "
                     f"steps, 8 workers, 32 executors, max 8 aggregated, median of {repeats}"}
    finals = set()
    ms = {mode: [] for mode in IntegrationMode}
    for _ in range(repeats):            # the modes' runs interleaved
        for mode in IntegrationMode:
            per, U = run_native_hydro(I, steps, workers=8, executors=32, max_agg=8, mode=mode)
            ms[mode].append(statistics.fmean(m.wall_ms for m in per[2:]))
            finals.add(hash(U.tobytes()))
            out[f"{mode.value}_mean_batch"] = per[-1].mean_batch
    for mode in IntegrationMode:
        out[f"{mode.value}_ms_per_step"] = statistics.median(ms[mode])
    out["speedup_polling_vs_fence"] = out["fence_ms_per_step"] / out["polling_ms_per_step"]
    out["speedup_hosttask_vs_fence"] = out["fence_ms_per_step"] / out["hosttask_ms_per_step"]
    out["results_identical"] = len(finals) == 1
    return out


def star_dist_bench(dev, rank, world, L=5, steps=5):
    """The rotating-star step at max_level 5 split into z-slabs over the
    job's ranks (StarSlab + DistDriver: NCCL halo planes of state and
    multipole records, all-gathered coarse level, MIN-reduced dt); strong
    scaling, CUDA events, max over ranks. Parity unpinned; bit-identical to
    the single-device step (tests/test_gpu_star_dist.py)."""
    import torch
    import torch.distributed as dist
    from paper_2303_08058_b200.hydro import rotating_star
    from paper_2303_08058_b200.star import subgrids_to_lattice
    from paper_2303_08058_b200.star_dist import DistDriver, StarSlab, split_state
    U = subgrids_to_lattice(rotating_star(8 ** L, device=dev)[0])
    slab = StarSlab(L, world, rank, split_state(U, world)[rank])
    del U
    drv = DistDriver(slab)
    for _ in range(2):
        drv.step()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        drv.step()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    cells = (8 << L) ** 3
    backend = dist.get_backend()
    return {"config": f"rotating-star step, max_level {L} ({cells} cells) in {world} z-slabs "
                      f"(one per rank, {backend}): halo planes of the state and of each "
                      "partitioned FMM level's multipole records, all-gathered coarse level, "
                      "MIN dt" + ("" if backend == "nccl" else
                                  " [non-NCCL: host-staged code-path test, not a timing]"),
            "ms_per_step": ms, "cells_per_s": cells / (ms * 1e-3), "scaling": "strong",
            "n_gpus": world,
            "parity": "unpinned (self-authored spec); bit-identical to the one-device step"}


def run_reference_arm(args, workload_key, rank, world):
    if rank != 0:
        return 0
    per_gpu, desc = WORKLOADS[workload_key]
    subgrids = per_gpu * world
    import numpy as np
    from oracle import c_oracle
    threads = len(os.sched_getaffinity(0))
    old = c_oracle.init_cells(subgrids)
    new = np.empty_like(old)
    mins, sums = np.empty(subgrids), np.empty(subgrids)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        c_oracle.step(old, new, old[-1, -8:].copy(), old[0, :8].copy(), mins, sums,
                      threads=threads)
        c_oracle.fsum(sums)
        float(mins.min())
        el = time.perf_counter() - t0
        old, new = new, old
        if i >= args.warmup:
            times.append(el)
    sec = sum(times) / len(times)
    value = subgrids * 512 / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "cells/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (closed-form ring ICs)",
        "config": {"workload": desc, "subgrids": subgrids, "cells": subgrids * 512,
                   "parallelism": f"cpu-openmp-{threads}t"},
        "cpu_baseline": {"value": value, "unit": "cells/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{args.steps} full steps of {subgrids} sub-grids "
                                   "(oracle/tb_oracle.c: C port of "
                                   "pkg/src/taskbridge/reference.py:23-50)"},
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[1])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c4")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-budget", type=float, default=10.0,
                    help="seconds of CPU work for the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--step-impl", choices=["auto", "reg", "bulk", "regpf", "lean", "pair", "bulk1"], default="auto",
                    help="K2 variant (tb_set_option TB_OPT_STEP_IMPL)")
    ap.add_argument("--e2e-chunks", type=int, default=8)
    ap.add_argument("--dist-backend", default="nccl",
                    help="torch.distributed backend for N>1 (gloo only to exercise the "
                         "multi-rank code path with several ranks on one GPU)")
    ap.add_argument("--halo", choices=["auto", "p2p", "nccl"], default="auto",
                    help="N>1 ring halo + reduction: p2p = neighbour faces and the exact "
                         "all-reduce over CUDA-IPC peer memory; nccl = NCCL send/recv of the "
                         "faces + NCCL all-reduces; auto = p2p when every rank can map its "
                         "neighbours, else nccl")
    ap.add_argument("--same-gpu", action="store_true",
                    help="all ranks on cuda:0 (with --dist-backend gloo: code-path test)")
    ap.add_argument("--no-ablation", action="store_true",
                    help="skip the polling/host-task/fence machine ablation")
    ap.add_argument("--no-kernels", action="store_true",
                    help="skip the hydro (K6) / FMM (K7) lines of configs 2 and 3")
    ap.add_argument("--warm-ms", type=float, default=20.0,
                    help="minimum device time of back-to-back warm-up steps before the "
                         "timed region (after the --warmup steps): long enough to leave "
                         "the idle power state, short of the ~100 ms of K2 load after "
                         "which sw_power_cap lowers SM clocks (profiles/r02/warmup_sweep.txt)")
    ap.add_argument("--spw", type=int, default=0,
                    help="K2 sub-grids per warp per CTA (0 = one persistent wave)")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    if args.same_gpu:
        local = 0
    if args.impl == "reference":
        return run_reference_arm(args, args.workload, rank, world)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            # the communicator's init lines (ranks, devices, transport) on
            # stderr, so the run shows NCCL formed the N-rank clique
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
            dist.barrier()          # eager communicator creation
        else:   # code-path testing only (several ranks sharing one GPU)
            dist.init_process_group(args.dist_backend)

    from paper_2303_08058_b200 import _native as N
    from paper_2303_08058_b200.ring import RingStepper, run_reference_gpu
    N.init(local)
    N.call("tb_set_option", N.TB_OPT_STEP_IMPL,
           {"auto": N.TB_STEP_AUTO, "reg": N.TB_STEP_REG, "bulk": N.TB_STEP_BULK,
            "regpf": N.TB_STEP_REGPF, "lean": N.TB_STEP_LEAN,
            "pair": N.TB_STEP_PAIR, "bulk1": N.TB_STEP_BULK1}[args.step_impl])
    N.call("tb_set_option", N.TB_OPT_STEP_SPW, args.spw)

    # Parity gate in the same run: the reference's GOLDEN_DEFAULTS.
    parity = run_reference_gpu(512, 15, device=dev)[0] == GOLDEN_DEFAULTS

    per_gpu, desc = WORKLOADS[args.workload]
    subgrids = per_gpu * world
    # (+ 4 scenario runs of SCENARIO_STEPS for e2e_scenario)
    total_steps = (args.warmup + args.steps + min(args.steps, 200) + args.e2e_steps + 8
                   + (4 * SCENARIO_STEPS if args.e2e_steps > 0 else 0)
                   + int(args.warm_ms / 0.02) + 128)     # time-based warm-up steps
    st = RingStepper(subgrids, device=dev, rank=rank, world=world, max_steps=total_steps,
                     group=None, halo=args.halo)
    n_local = st.n
    # Warm-up: W steps, then more back-to-back steps until >= --warm-ms of
    # device time has run, ending right before the timed region with no idle
    # gap. After an idle gap the first steps run slow (profiles/r02/
    # k2_trace.json: 140, 72, then 53 us); after >= ~100 ms of back-to-back
    # K2 the board reaches sw_power_cap and SM clocks fall to ~1780 MHz
    # (profiles/r02/warmup_sweep.txt) — the default 20 ms sits between.
    # Declared in the line as "warmup_policy".
    sampler = ClockSampler(local)
    sampler.start()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    warm_steps = 0
    while warm_steps < args.warmup or time.perf_counter() - w0 < args.warm_ms * 1e-3:
        k = max(1, min(args.warmup - warm_steps, 64)) if warm_steps < args.warmup else 32
        for _ in range(k):
            st.step()
        warm_steps += k
        if warm_steps >= args.warmup:
            torch.cuda.synchronize()
    warm_ms = (time.perf_counter() - w0) * 1e3
    # Headline: K steps back to back, no L2 flush. Each step reads the
    # previous step's 128 MiB output (> the 126 MB L2) from the start while
    # its tail is the most recently written, so nothing is re-read from L2
    # (ncu --cache-control none: profiles/r01_k2_back_to_back.txt). N = 1:
    # one launch per step, so the outer events time K2; N > 1: K2 is
    # bracketed per step.
    per_step_k2 = world > 1
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps if per_step_k2 else 0)]
    e_start, e_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.edges["before"] = sampler.sample()
    t_wall = time.perf_counter()
    e_start.record()
    for i in range(args.steps):
        st.step(kernel_events=ev[i] if per_step_k2 else None)
    timed_launches = (1 if world == 1 else 2) * args.steps
    e_stop.record()
    while not e_stop.query():        # the launches are asynchronous: sample under load
        sampler.sample(sampler.during)
    torch.cuda.synchronize()
    t_end = time.perf_counter()
    wall = t_end - t_wall
    sampler.window = (t_wall, t_end)
    sampler.edges["after"] = sampler.sample()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = e_start.elapsed_time(e_stop) / args.steps
    k2_ms = (sum(a.elapsed_time(b) for a, b in ev) / args.steps) if per_step_k2 else step_ms
    # Secondary: the same step with a 256 MiB L2-flushing write before every
    # step, events per step (the conservative cold-cache number).
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    kf = min(args.steps, 200)
    evf = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(kf)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for (s0, s1, k0, k1) in evf:
        flush.fill_(1)
        s0.record()
        st.step(kernel_events=(k0, k1))
        s1.record()
    torch.cuda.synchronize()
    flushed_step_ms = sum(a.elapsed_time(b) for a, b, _, _ in evf) / kf
    flushed_k2_ms = sum(c.elapsed_time(d) for _, _, c, d in evf) / kf
    if world > 1:
        t = torch.tensor([step_ms, k2_ms, flushed_step_ms, flushed_k2_ms], dtype=torch.float64,
                         device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms, k2_ms, flushed_step_ms, flushed_k2_ms = t.tolist()
    cells_total = subgrids * 512
    # back-to-back timing is only valid when a step's input exceeds the L2
    # (C4, C5); smaller rings (C2: 16 MiB) take the flushed per-step numbers
    l2_bytes = 126e6
    b2b_valid = n_local * 512 * 8 > l2_bytes
    if not b2b_valid:
        step_ms, k2_ms = flushed_step_ms, flushed_k2_ms
    value = cells_total / (step_ms * 1e-3)

    # ---- e2e through the host-buffer API (pinned H2D + step + D2H) ------
    e2e = None
    if args.e2e_steps > 0:
        host_in = torch.empty((n_local, 512), dtype=torch.float64, pin_memory=True)
        host_in.copy_(st.cells)
        host_stats = torch.empty(2, dtype=torch.float64, pin_memory=True)
        for _ in range(2):     # warm the copy streams / events / pinned-copy paths
            st.step_host(host_in, host_in, host_stats, chunks=args.e2e_chunks)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.e2e_steps):
            st.step_host(host_in, host_in, host_stats, chunks=args.e2e_chunks, join=False)
        st.join_host()
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = t.item()
        e2e = {"value": cells_total / (e2e_ms * 1e-3), "unit": "cells/s",
               "h2d_bytes_per_step": n_local * 512 * 8,
               "d2h_bytes_per_step": n_local * 512 * 8 + 16,
               "ms_per_step": e2e_ms, "chunks": args.e2e_chunks,
               "api": "RingStepper.step_host (pinned H2D | K2 | D2H pipelined "
                      "over chunks on 3 streams, chained across steps)"}

        # the same public API at the reference's call granularity: one
        # run_scenario-style call = cells H2D from pinned host memory,
        # SCENARIO_STEPS steps resident in HBM, (checksum, dts) and the final
        # cells D2H — the copies amortised over the call's steps
        host_out = torch.empty((n_local, 512), dtype=torch.float64, pin_memory=True)
        runs = []
        for r in range(4):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            st.load_cells(host_in)
            if world > 1:       # peer-memory halos read the neighbours' new cells
                torch.cuda.synchronize()
                dist.barrier()
            st.run(SCENARIO_STEPS)                  # reads (checksum, dts) back
            host_out.copy_(st.cells, non_blocking=True)
            b.record()
            torch.cuda.synchronize()
            if r:                                   # the first call warms up
                runs.append(a.elapsed_time(b))
        run_ms = sum(runs) / len(runs)
        if world > 1:
            t = torch.tensor([run_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            run_ms = t.item()
        e2e["scenario_call"] = {
            "value": cells_total * SCENARIO_STEPS / (run_ms * 1e-3), "unit": "cells/s",
            "steps_per_call": SCENARIO_STEPS, "ms_per_call": run_ms,
            "h2d_bytes_per_step": n_local * 512 * 8 / SCENARIO_STEPS,
            "d2h_bytes_per_step": (n_local * 512 * 8 + 16 * SCENARIO_STEPS + 8) / SCENARIO_STEPS,
            "api": "RingStepper.load_cells(pinned host) + run(15) + cells to pinned host "
                   "(run_scenario's call granularity; the headline e2e above copies every step)"}

        if world == 1 and not args.no_ablation:
            e2e["plugin_call"] = plugin_call_bench()

    star_dist = None
    if world > 1 and not args.no_kernels:
        # a failure here must not cost the headline line (local errors, e.g.
        # a slab geometry the rank count does not divide, raise before any
        # collective of the step)
        try:
            star_dist = star_dist_bench(dev, rank, world)
        except Exception as e:  # noqa: BLE001
            star_dist = {"error": f"{type(e).__name__}: {e}"[:300]}
    if rank == 0:
        peaks, peak_kind = measured_peaks()
        hbm = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
        achieved = n_local * 512 * BYTES_PER_CELL / (k2_ms * 1e-3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "k2_traffic.json")
        if os.path.exists(tpath):
            try:
                with open(tpath) as fh:
                    tj = json.load(fh)
                impl_key = AUTO_IMPL if args.step_impl == "auto" else args.step_impl
                ent = tj.get("by_impl", {}).get(impl_key)
                if ent and tj.get("subgrids") == n_local:
                    traffic = ent["dram_bytes_per_launch"]
            except (OSError, ValueError, KeyError):
                pass
        ablation = None
        if not args.no_ablation:
            ablation = machine_ablation()
            ablation["c4"] = machine_ablation_c4()
            ablation["hydro_machine"] = hydro_machine_ablation()
        kernels = None
        if not args.no_kernels:
            kernels = north_star_kernels(dev)
            if star_dist is not None:
                kernels["star_step_dist"] = star_dist
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            v, cores, nsteps, el = cpu_reference_sample(per_gpu, args.cpu_budget)
            cpu = {"value": v, "unit": "cells/s", "cores": cores, "kind": "port",
                   "sample": f"{nsteps} full steps of {per_gpu} sub-grids in {el:.1f}s "
                             "(oracle/tb_oracle.c, OpenMP)",
                   "python_reference": python_reference_sample()}
        line = {
            "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (closed-form ring ICs, src/miniapp.py:72-77)",
            "config": {"workload": desc, "subgrids": subgrids, "subgrids_per_gpu": per_gpu,
                       "cells": cells_total, "parallelism": f"ring-dp{world}",
                       "halo": st.halo_mode,
                       "reduction": ("peer-memory atomics (tb_acc_allreduce_p2p)"
                                     if st.halo_mode == "p2p" else
                                     ("nccl all_reduce" if world > 1 else "in-kernel")),
                       "l2": ("no flush: steps back to back, inputs larger than L2 (each "
                              "step reads the previous step's 128 MiB output; 126 MB L2; ncu "
                              "--cache-control none: 135 MB DRAM reads per launch = the whole "
                              "input, profiles/r01_k2_back_to_back.txt); the flushed number "
                              "is l2_flushed_per_step") if b2b_valid else
                             ("flushed: a 256 MiB write before every timed step, events per "
                              "step (the state fits in L2, so back-to-back timing would "
                              "measure L2)")},
            "l2_flushed_per_step": {
                "ms_per_step": flushed_step_ms, "value": cells_total / (flushed_step_ms * 1e-3),
                "k2_ms": flushed_k2_ms,
                "k2_frac": n_local * 512 * BYTES_PER_CELL / (flushed_k2_ms * 1e-3) / 1e9 / hbm,
                "method": "256 MiB write before every timed step, CUDA events per step"},
            "parity": {"run_reference_512x15_equals_GOLDEN_DEFAULTS": parity},
            "roofline": {"bound": "hbm",
                         "kernel": {"auto": "k_step_bulk<3,5,1 stage>",
                               "bulk": "k_step_bulk<3,5>",
                               "reg": "k_step<3,5>", "regpf": "k_step<3,5,pf>",
                               "lean": "k_step<3,5,lean48>",
                               "pair": "k_step_pair<3,5>",
                               "bulk1": "k_step_bulk<3,5,1 stage>"}[
                                   args.step_impl] + (
                                       " (tb_step_deferred: K2, the previous step's "
                                       "exact close in its extra CTA)"
                                       if world == 1 else " (tb_step)"),
                         "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm,
                         "traffic": traffic,
                         "traffic_note": "ncu dram__bytes_read+write per K2 launch "
                                         "(profiles/k2_traffic.json)",
                         "algorithmic_bytes_per_launch": n_local * 512 * BYTES_PER_CELL,
                         "peak_source": peak_kind,
                         "bytes_per_cell": BYTES_PER_CELL, "k2_ms": k2_ms,
                         # the co-limit: 15 x (DMUL + DADD) + fold
                         # + pairwise sum + min, FMA forbidden by parity
                         "fp64": {"instr_per_cell": FP64_PER_CELL,
                                  "achieved": FP64_PER_CELL * n_local * 512 / (k2_ms * 1e-3),
                                  "peak": fp64_peak()[0], "peak_source": fp64_peak()[1],
                                  "unit": "FP64 instr/s",
                                  "frac": FP64_PER_CELL * n_local * 512 / (k2_ms * 1e-3)
                                  / fp64_peak()[0]}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "ablation": ablation,
            "north_star_kernels": kernels,
            "gpu_launches": timed_launches,
            "warmup_policy": {"steps": warm_steps, "min_ms": args.warm_ms,
                              "ms": warm_ms,
                              "rule": "--warmup steps, then back-to-back steps until "
                                      "--warm-ms of device time, immediately before the "
                                      "timed region (synchronize, no idle gap); longer "
                                      "warm-ups reach sw_power_cap (profiles/r02/"
                                      "warmup_sweep.txt)"},
            "clocks": clocks,
            "wall_s_timed_region": wall,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
