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
        "hosttask_threads", "zero_copy", "fault_at_launch", "completion")]


_COMPLETION = {"events": N.TB_COMPLETION_EVENTS, "words": N.TB_COMPLETION_WORDS}


class MachineStep(ctypes.Structure):
    _fields_ = [("wall_ms", ctypes.c_double), ("dt", ctypes.c_double),
                ("piece", ctypes.c_double)] + [
        (name, ctypes.c_int64) for name in (
            "launches", "transfers", "event_waits", "full", "idle", "members")]


ZERO_COPY_GATHER = 2


def run_native(subgrids: int, steps: int, workers: int = 8, executors: int = 32,
               max_agg: int = 8, mode: IntegrationMode = IntegrationMode.POLLING,
               inject_barriers: bool = True, barrier_elision: bool = False,
               task_subgrids: int = 1, hosttask_threads: int = 2, device: int = 0,
               chains: int = 3, kernels_per_chain: int = 5,
               return_cells: bool = False, zero_copy=False, fault_at_launch: int = 0,
               cells: Optional[np.ndarray] = None, exec_stats: Optional[np.ndarray] = None,
               completion: str = "events"):
    """Run the machine natively; returns (ScenarioResult, cells or None).

    ``zero_copy``: False/0 = the reference op sequence per batch (H2D ;
    kernel ; D2H); True/1 = the batch kernel works in place on its pinned
    staging buffer; 2 (ZERO_COPY_GATHER) = no staging: the tasks' buffers
    live in pinned memory and the batch kernel reads and writes each member
    where it lives; 3 = gather with each task's rounds between the first and
    the last in device memory; 4 = direct: 3 without any host copy of the
    cells — the first round's kernel reads the rows and folds the neighbour
    faces, the last writes them back with their min and pairwise sum (the
    rows must be pinned, mapped host memory: ``cells`` from a pinned
    allocation, or the machine's own). ``cells`` ([subgrids, 512] float64, C-contiguous):
    start from (and write the final state back into) these cells instead of
    the closed-form initial state. ``fault_at_launch`` (tests): the k-th
    batch launch traps; the device fault surfaces as a raised CudaError.
    ``completion``: "events" (a CUDA event per batch and probe, queried /
    synchronized / called back) or "words" (zero_copy >= 2, POLLING or
    FENCE: the batch kernel stores its sequence number in the executor's
    mapped completion word; polling and fencing read memory).
    ``exec_stats`` (with ``cells``): int64 [steps, executors, max_agg + 3]
    receiving per-executor batch-size histograms and full/idle counts."""
    N.init(device)
    cfg = MachineConfig(subgrids, steps, chains, kernels_per_chain, workers, executors,
                        max_agg, _MODES[mode], int(inject_barriers), int(barrier_elision),
                        task_subgrids, hosttask_threads, int(zero_copy), int(fault_at_launch),
                        _COMPLETION[completion])
    out = (MachineStep * max(steps, 1))()
    cs = ctypes.c_double(0.0)
    if cells is not None:
        if (cells.dtype != np.float64 or cells.shape != (subgrids, 512)
                or not cells.flags.c_contiguous or not cells.flags.writeable):
            raise ValueError("cells must be a writable C-contiguous float64 [subgrids, 512]")
        if exec_stats is not None and (exec_stats.dtype != np.int64 or exec_stats.shape != (
                steps, executors, max_agg + 3) or not exec_stats.flags.c_contiguous):
            raise ValueError("exec_stats must be C-contiguous int64 [steps, executors, max_agg+3]")
        N.call("tb_machine_run_cells", ctypes.addressof(cfg), cells.ctypes.data,
               ctypes.addressof(cs), ctypes.addressof(out),
               None if exec_stats is None else exec_stats.ctypes.data)
    else:
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
                          dts=[o.dt for o in out[:steps]], engine="native"), cells


def run_native_hydro(state: np.ndarray, steps: int, workers: int = 8, executors: int = 32,
                     max_agg: int = 8, mode: IntegrationMode = IntegrationMode.POLLING,
                     task_subgrids: int = 1, hosttask_threads: int = 2, device: int = 0,
                     cfl: float = 0.4, gamma: float = 5.0 / 3.0, fault_at_launch: int = 0):
    """The machine on the north_star's hydro kernel (tb_machine_run_hydro):
    per step one task per ``task_subgrids`` sub-grids does the periodic ghost
    exchange on the host and schedules an aggregated K6 request; completion
    by ``mode``; then the forward-Euler update. ``state``: [S, 5, 8, 8, 8]
    float64 (S = n^3). Returns (per-step StepMetrics, final state)."""
    N.init(device)
    st = np.ascontiguousarray(state, dtype=np.float64)
    S = st.shape[0]
    cfg = MachineConfig(S, steps, 0, 1, workers, executors, max_agg, _MODES[mode], 0, 0,
                        task_subgrids, hosttask_threads, 0, int(fault_at_launch))
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
