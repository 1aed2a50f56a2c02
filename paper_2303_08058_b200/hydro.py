"""Hydro reconstruct-and-flux on the GPU (K6, ``tb_hydro_flux``).

The north_star's "hydro reconstruct+flux only on a batch of 4096 synthetic
8^3 sub-grids with ghost layers" (BASELINE.json config 2). PARITY UNPINNED:
the reference has no hydro; the arithmetic follows the
self-authored spec in ``oracle/hydro_oracle.py`` bit for bit.

Layout: U [S, 5, 12, 12, 12] float64 (rho, sx, sy, sz, E; 2-cell ghost
layers), dU/dt [S, 5, 8, 8, 8], amax [S].
"""

from __future__ import annotations

from typing import Optional, Tuple

import torch

from . import _native as N

NG, NI, NT, NF = 2, 8, 12, 5


def hydro_flux(U: torch.Tensor, dx: float, gamma: float = 5.0 / 3.0,
               out: Optional[torch.Tensor] = None,
               amax: Optional[torch.Tensor] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """dU/dt of every interior cell and the per-sub-grid max signal speed."""
    if U.device.type != "cuda":
        raise RuntimeError("hydro_flux needs a CUDA tensor (no CPU fallback)")
    if U.dtype != torch.float64 or tuple(U.shape[1:]) != (NF, NT, NT, NT):
        raise ValueError("U must be float64 [S, 5, 12, 12, 12]")
    U = U.contiguous()
    s = U.shape[0]
    if out is None:
        out = torch.empty((s, NF, NI, NI, NI), dtype=torch.float64, device=U.device)
    if amax is None:
        amax = torch.empty(s, dtype=torch.float64, device=U.device)
    N.init(U.device.index or 0)
    N.call("tb_hydro_flux", torch.cuda.current_stream(U.device).cuda_stream, U.data_ptr(),
           out.data_ptr(), amax.data_ptr(), s, float(dx), float(gamma))
    return out, amax


# ------------------------------------------------------- synthetic inputs --
def rotating_star(subgrids: int, gamma: float = 5.0 / 3.0, omega: float = 0.3,
                  device=None) -> Tuple[torch.Tensor, float]:
    """Synthetic rotating star on a periodic lattice of n^3 sub-grids in the
    unit cube (a polytrope-like density bump in solid-body rotation about z
    on a low floor). Returns (interior state [n^3, 5, 8, 8, 8] float64, dx);
    sub-grid order x fastest. Same numbers as the oracle's generator
    (tests/test_hydro_oracle.py checks it)."""
    n = round(subgrids ** (1.0 / 3.0))
    if n ** 3 != subgrids:
        raise ValueError("subgrids must be a cube (a uniform octree level)")
    N = n * NI
    dx = 1.0 / N
    c = (torch.arange(N, dtype=torch.float64, device=device) + 0.5) * dx - 0.5
    z, y, x = torch.meshgrid(c, c, c, indexing="ij")
    r = torch.sqrt(x * x + y * y + z * z)
    rho = 1e-3 + torch.clamp(1.0 - (r / 0.35) ** 2, min=0.0) ** 1.5
    vx, vy, vz = -omega * y, omega * x, torch.zeros_like(x)
    p = 1e-4 + 0.3 * rho ** gamma
    E = p / (gamma - 1.0) + 0.5 * rho * (vx * vx + vy * vy + vz * vz)
    glob = torch.stack([rho, rho * vx, rho * vy, rho * vz, E])        # [5, N, N, N]
    g = glob.reshape(NF, n, NI, n, NI, n, NI).permute(1, 3, 5, 0, 2, 4, 6)
    return g.reshape(subgrids, NF, NI, NI, NI).contiguous(), dx


def with_ghosts(interior: torch.Tensor) -> torch.Tensor:
    """Fill the 2-cell ghost layers of every sub-grid from its periodic
    lattice neighbours -> [S, 5, 12, 12, 12] (what the octree's ghost
    exchange provides)."""
    s = interior.shape[0]
    n = round(s ** (1.0 / 3.0))
    N = n * NI
    glob = interior.reshape(n, n, n, NF, NI, NI, NI).permute(3, 0, 4, 1, 5, 2, 6)
    glob = glob.reshape(1, NF, N, N, N)
    pad = torch.nn.functional.pad(glob, (NG,) * 6, mode="circular")[0]   # [5, N+4, ...]
    blocks = pad.unfold(1, NT, NI).unfold(2, NT, NI).unfold(3, NT, NI)   # [5,n,n,n,12,12,12]
    return blocks.permute(1, 2, 3, 0, 4, 5, 6).reshape(s, NF, NT, NT, NT).contiguous()
