"""FMM gravity on the GPU (K7, ``tb_fmm_*``).

The north_star's "FMM monopole/multipole stencil-interaction kernels"
(BASELINE.json config 3: "FMM multipole+monopole interaction kernels only,
rotating star max_level 4"). PARITY UNPINNED: the reference has no gravity
solver; the spec is the self-authored
``oracle/fmm_oracle.py``, matched per cell to 1e-10 relative.

Layout: rho [N, N, N] float64 (z, y, x; N = 8 * 2^max_level leaf cells per
edge of the unit cube, isolated boundary); result [4, N, N, N] =
(phi, gx, gy, gz), g = -grad phi, G = 1.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _native as N


def workspace_bytes(max_level: int) -> int:
    n = ctypes.c_uint64(0)
    N.call("tb_fmm_workspace_bytes", max_level, ctypes.byref(n))
    return n.value


class GravitySolver:
    """Uniform-octree FMM of depth ``max_level`` on one CUDA device. The
    workspace (per-level multipoles and local expansions) stays resident in
    HBM between solves; ``solve`` enqueues 2*max_level + 1 launches on the
    current stream."""

    def __init__(self, max_level: int, device: Optional[torch.device] = None):
        if max_level < 1:
            raise ValueError("max_level must be >= 1")
        self.max_level = max_level
        self.n = 8 << max_level
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        if self.device.type != "cuda":
            raise RuntimeError("GravitySolver needs a CUDA device (no CPU fallback)")
        N.init(self.device.index or 0)
        nbytes = workspace_bytes(max_level)
        # zeroed once: the halo planes of the partitioned levels' moment
        # records stay zero on one device (= the isolated boundary)
        self.work = torch.zeros(nbytes // 8, dtype=torch.float64, device=self.device)
        self.out = torch.empty((4, self.n, self.n, self.n), dtype=torch.float64,
                               device=self.device)

    def _check(self, rho: torch.Tensor) -> torch.Tensor:
        if rho.device != self.out.device or rho.dtype != torch.float64:
            raise ValueError("rho must be a float64 tensor on the solver's device")
        if tuple(rho.shape) != (self.n,) * 3:
            raise ValueError(f"rho must be [{self.n}]^3")
        return rho.contiguous()

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def upward(self, rho: torch.Tensor) -> None:
        N.call("tb_fmm_upward", self._stream(), self.max_level, rho.data_ptr(),
               self.work.data_ptr())

    def m2l(self) -> None:
        """Multipole interactions of every level (one launch)."""
        N.call("tb_fmm_m2l", self._stream(), self.max_level, self.work.data_ptr())

    def downward(self) -> None:
        N.call("tb_fmm_downward", self._stream(), self.max_level, self.work.data_ptr())

    def leaf(self, rho: torch.Tensor) -> torch.Tensor:
        """Monopole interactions at the leaves + L2P -> (phi, gx, gy, gz)."""
        N.call("tb_fmm_leaf", self._stream(), self.max_level, rho.data_ptr(),
               self.work.data_ptr(), self.out.data_ptr())
        return self.out

    def solve(self, rho: torch.Tensor) -> torch.Tensor:
        rho = self._check(rho)
        N.call("tb_fmm_solve", self._stream(), self.max_level, rho.data_ptr(),
               self.work.data_ptr(), self.out.data_ptr())
        return self.out


def fmm_gravity(rho: torch.Tensor, max_level: Optional[int] = None) -> torch.Tensor:
    """One-shot solve: returns a new [4, N, N, N] tensor."""
    n = rho.shape[0]
    lev = max_level if max_level is not None else (n // 8).bit_length() - 1
    s = GravitySolver(lev, rho.device)
    return s.solve(rho).clone()


def rotating_star_density(max_level: int, device=None) -> torch.Tensor:
    """The synthetic rotating star's density (the hydro generator's bump on a
    1e-3 floor) as an [N, N, N] leaf lattice, N = 8 * 2^max_level, on the
    isolated unit cube (tests check it against the oracle's generator)."""
    N = 8 << max_level
    c = (torch.arange(N, dtype=torch.float64, device=device) + 0.5) / N - 0.5
    z, y, x = torch.meshgrid(c, c, c, indexing="ij")
    r = torch.sqrt(x * x + y * y + z * z)
    return (1e-3 + torch.clamp(1.0 - (r / 0.35) ** 2, min=0.0) ** 1.5).contiguous()
