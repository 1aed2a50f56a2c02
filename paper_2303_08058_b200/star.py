"""The coupled rotating-star step on the GPU: hydro (K6) + FMM gravity (K7)
+ SSP-RK2, device-resident (the north_star's "full rotating-star step").

PARITY UNPINNED: the reference has no physics; the spec is
the self-authored ``oracle/star_oracle.py``, matched per cell to 1e-10.

One step = 2 x [periodic ghost pad -> hydro flux (4-D TMA boxes from the
padded lattice) -> FMM solve of rho -> RK stage] + the CFL dt, all enqueued on
one stream with dt kept in device memory (no host round trip). ``graph=True``
captures the whole step once in a CUDA graph and replays it.
"""

from __future__ import annotations

from typing import Optional

import torch

from . import _native as N
from .gravity import GravitySolver
from .hydro import NF, NI, rotating_star


def subgrids_to_lattice(S: torch.Tensor) -> torch.Tensor:
    """[n^3, F, 8, 8, 8] -> [F, N, N, N]."""
    s, F = S.shape[:2]
    n = round(s ** (1 / 3))
    g = S.reshape(n, n, n, F, NI, NI, NI).permute(3, 0, 4, 1, 5, 2, 6)
    return g.reshape(F, n * NI, n * NI, n * NI).contiguous()


class RotatingStarStep:
    """SSP-RK2 time stepper of the rotating star at ``max_level`` (lattice
    N = 8 * 2^max_level per edge) on one CUDA device."""

    def __init__(self, max_level: int, gamma: float = 5.0 / 3.0, cfl: float = 0.4,
                 omega: float = 0.3, device: Optional[torch.device] = None,
                 state: Optional[torch.Tensor] = None, concurrent: bool = True,
                 record_stages: bool = False):
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        if self.device.type != "cuda":
            raise RuntimeError("RotatingStarStep needs a CUDA device (no CPU fallback)")
        N.init(self.device.index or 0)
        self.max_level, self.gamma, self.cfl = max_level, float(gamma), float(cfl)
        self.n = 8 << max_level
        self.nsub = (self.n // NI) ** 3
        self.dx = 1.0 / self.n
        if state is None:
            I, _ = rotating_star(self.nsub, gamma, omega, device=self.device)
            state = subgrids_to_lattice(I)
        if tuple(state.shape) != (NF, self.n, self.n, self.n) or state.dtype != torch.float64:
            raise ValueError("state must be float64 [5, N, N, N]")
        f64 = dict(dtype=torch.float64, device=self.device)
        self.U = state.to(self.device).contiguous().clone()
        self.U1 = torch.empty_like(self.U)
        p = self.n + 4
        self.Up = torch.empty((NF, p, p, p), **f64)
        self.dudt = torch.empty((self.nsub, NF, NI, NI, NI), **f64)
        self.amax = torch.empty(self.nsub, **f64)
        self.dt = torch.zeros(1, **f64)
        self.time = torch.zeros(1, **f64)
        self.gravity = GravitySolver(max_level, self.device)
        self._graph = None
        self._concurrent = concurrent
        self._side = torch.cuda.Stream(self.device) if concurrent else None
        # verification mode (tests): keep the stage-1 per-sub-grid amax and
        # both stages' g (the step itself overwrites them); costs 3 copies
        self.record_stages = record_stages
        if record_stages:
            self.amax1 = torch.empty_like(self.amax)
            self.g1 = torch.empty((3, self.n, self.n, self.n), **f64)
            self.g2 = torch.empty_like(self.g1)

    def _s(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def _rhs(self, Uc: torch.Tensor) -> None:
        # hydro (pad + K6) and gravity (K7) both only read Uc: the hydro
        # branch runs on a side stream so it fills the SMs the FMM's coarse
        # levels leave idle (fork/join by events; captured as graph branches)
        main = torch.cuda.current_stream(self.device)
        if self._concurrent:
            self._side.wait_stream(main)
            s = self._side.cuda_stream
        else:
            s = main.cuda_stream
        N.call("tb_star_pad", s, Uc.data_ptr(), self.n, self.Up.data_ptr())
        N.call("tb_hydro_flux_lattice", s, self.Up.data_ptr(), self.n, self.n,
               self.dudt.data_ptr(), self.amax.data_ptr(), self.dx, self.gamma)
        self.gravity.solve(Uc[0])
        if self._concurrent:
            main.wait_stream(self._side)

    def _g(self) -> int:
        return self.gravity.out.data_ptr() + self.n ** 3 * 8     # rows 1..3 of [4][N^3]

    def _gview(self) -> torch.Tensor:
        return self.gravity.out[1:4].reshape(3, self.n, self.n, self.n)

    def _enqueue_step(self) -> None:
        s = self._s()
        self._rhs(self.U)
        if self.record_stages:
            self.amax1.copy_(self.amax)
            self.g1.copy_(self._gview())
        N.call("tb_star_cfl", s, self.amax.data_ptr(), self.nsub, self.dx, self.cfl,
               self.dt.data_ptr())
        N.call("tb_star_stage", s, 1, None, self.U.data_ptr(), self.dudt.data_ptr(), self._g(),
               self.dt.data_ptr(), self.n, self.n, self.U1.data_ptr())
        self._rhs(self.U1)
        if self.record_stages:
            self.g2.copy_(self._gview())
        N.call("tb_star_stage", s, 2, self.U.data_ptr(), self.U1.data_ptr(),
               self.dudt.data_ptr(), self._g(), self.dt.data_ptr(), self.n, self.n,
               self.U.data_ptr())
        self.time.add_(self.dt)

    def step(self, graph: bool = False) -> None:
        """Advance one step (asynchronously; ``self.dt`` / ``self.time`` stay
        on the device)."""
        if not graph:
            self._enqueue_step()
            return
        if self._graph is None:
            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):          # warm-up outside capture
                u, t = self.U.clone(), self.time.clone()
                self._enqueue_step()
                self.U.copy_(u)
                self.time.copy_(t)
            torch.cuda.current_stream(self.device).wait_stream(side)
            self._graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self._graph):
                self._enqueue_step()
        self._graph.replay()

    def launches_per_step(self) -> int:
        """Kernels one step launches (2 x (pad, hydro, 2L+3 FMM, stage) + cfl)."""
        return 2 * (2 + (2 * self.max_level + 3) + 1) + 1

    def totals(self):
        """(mass, momentum[3], energy) — conserved sums (host sync)."""
        t = self.U.sum(dim=(1, 2, 3)) * self.dx ** 3
        return t[0].item(), t[1:4].tolist(), t[4].item()
