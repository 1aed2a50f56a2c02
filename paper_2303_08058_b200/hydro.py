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
