"""ctypes front of ``tb_machine_run`` (include/tb.h): the reference machine
(src/cli.py:199-232 run_single) executed by libtb's native C++ runtime —
work-stealing workers that poll CUDA events between tasks (or complete them
from host-task threads, or fence), per-stream aggregation executors, and the
mini-app step driver. Returns the same ScenarioResult as
:func:`paper_2303_08058_b200.miniapp.run_scenario`.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _native as N
from .bridge import IntegrationMode
from .miniapp import ScenarioResult, StepMetrics

_MODES = {IntegrationMode.POLLING: N.TB_MODE_POLLING,
          IntegrationMode.HOSTTASK: N.TB_MODE_HOSTTASK,
          IntegrationMode.FENCE: N.TB_MODE_FENCE}


class MachineConfig(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "subgrids", "steps", "chains", "kernels_per_chain", "workers", "executors",
        "max_agg", "mode", "inject_barriers", "barrier_elision", "task_subgrids",
        "hosttask_threads", "zero_copy")]


class MachineStep(ctypes.Structure):
    _fields_ = [("wall_ms", ctypes.c_double), ("dt", ctypes.c_double),
                ("piece", ctypes.c_double)] + [
        (name, ctypes.c_int64) for name in (
            "launches", "transfers", "event_waits", "full", "idle", "members")]


def run_native(subgrids: int, steps: int, workers: int = 8, executors: int = 32,
               max_agg: int = 8, mode: IntegrationMode = IntegrationMode.POLLING,
               inject_barriers: bool = True, barrier_elision: bool = False,
               task_subgrids: int = 1, hosttask_threads: int = 2, device: int = 0,
               chains: int = 3, kernels_per_chain: int = 5,
               return_cells: bool = False, zero_copy: bool = False):
    """Run the machine natively; returns (ScenarioResult, cells or None).
    ``zero_copy``: each batch's kernel works in place on its pinned staging
    buffer (one launch + one event per batch instead of H2D ; kernel ; D2H)."""
    N.init(device)
    cfg = MachineConfig(subgrids, steps, chains, kernels_per_chain, workers, executors,
                        max_agg, _MODES[mode], int(inject_barriers), int(barrier_elision),
                        task_subgrids, hosttask_threads, int(zero_copy))
    out = (MachineStep * max(steps, 1))()
    cs = ctypes.c_double(0.0)
    cells: Optional[np.ndarray] = None
    if return_cells:
        cells = np.empty((subgrids, 512))
    N.call("tb_machine_run", ctypes.addressof(cfg), ctypes.addressof(cs),
           ctypes.addressof(out), None if cells is None else cells.ctypes.data)
    per_step = []
    for k in range(steps):
        o = out[k]
        per_step.append(StepMetrics(
            wall_ms=o.wall_ms, dt=o.dt, checksum_piece=o.piece, launches=o.launches,
            transfers=o.transfers, batch_sizes=[], reasons_full=o.full,
            reasons_idle=o.idle, event_waits=o.event_waits))
        per_step[-1].mean_batch = o.members / max(o.full + o.idle, 1)
    return ScenarioResult(per_step=per_step, checksum=cs.value,
                          dts=[o.dt for o in out[:steps]]), cells


def run_native_hydro(state: np.ndarray, steps: int, workers: int = 8, executors: int = 32,
                     max_agg: int = 8, mode: IntegrationMode = IntegrationMode.POLLING,
                     task_subgrids: int = 1, hosttask_threads: int = 2, device: int = 0,
                     cfl: float = 0.4, gamma: float = 5.0 / 3.0):
    """The machine on the north_star's hydro kernel (tb_machine_run_hydro):
    per step one task per ``task_subgrids`` sub-grids does the periodic ghost
    exchange on the host and schedules an aggregated K6 request; completion
    by ``mode``; then the forward-Euler update. ``state``: [S, 5, 8, 8, 8]
    float64 (S = n^3). Returns (per-step StepMetrics, final state)."""
    N.init(device)
    st = np.ascontiguousarray(state, dtype=np.float64)
    S = st.shape[0]
    cfg = MachineConfig(S, steps, 0, 1, workers, executors, max_agg, _MODES[mode], 0, 0,
                        task_subgrids, hosttask_threads)
    out = (MachineStep * max(steps, 1))()
    final = np.empty_like(st)
    N.call("tb_machine_run_hydro", ctypes.addressof(cfg), st.ctypes.data, final.ctypes.data,
           float(cfl), float(gamma), ctypes.addressof(out))
    per_step = []
    for k in range(steps):
        o = out[k]
        m = StepMetrics(wall_ms=o.wall_ms, dt=o.dt, checksum_piece=o.piece, launches=o.launches,
                        transfers=o.transfers, batch_sizes=[], reasons_full=o.full,
                        reasons_idle=o.idle, event_waits=o.event_waits)
        m.mean_batch = o.members / max(o.full + o.idle, 1)
        per_step.append(m)
    return per_step, final
