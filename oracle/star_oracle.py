"""numpy oracle for the coupled rotating-star step — TEST INFRASTRUCTURE.

PARITY UNPINNED: the reference has no physics. This is the
north_star's "full rotating-star step" as a SELF-AUTHORED spec composed of
the two self-authored kernels (oracle/hydro_oracle.py, oracle/fmm_oracle.py):

* state U [5, N, N, N] (rho, sx, sy, sz, E) on the unit cube, N = 8 * 2^L
  (the octree's leaf level), sub-grid s = (bz*n + by)*n + bx of 8^3 cells;
* hydro: periodic 2-cell ghost layers, dU/dt and per-sub-grid amax;
* gravity: FMM of rho with isolated boundary -> g;
* L(U) = dU/dt + (0, rho gx, rho gy, rho gz, (sx gx + sy gy) + sz gz);
* dt = (cfl * dx) / max(amax) from the stage-1 state;
* Heun / SSP-RK2: U1 = U + dt L(U);  U' = 0.5 * (U + (U1 + dt L(U1))).

Properties (tests/test_star_oracle.py): total mass conserved to round-off;
a uniform gas at rest stays at rest up to gravity; GPU per cell within 1e-10.
"""

from __future__ import annotations

import numpy as np

from . import fmm_oracle as fo
from . import hydro_oracle as ho

NF, NI = 5, 8


def subgrids_to_lattice(S: np.ndarray) -> np.ndarray:
    """[n^3, F, 8, 8, 8] -> [F, N, N, N]."""
    s, F = S.shape[:2]
    n = round(s ** (1 / 3))
    g = S.reshape(n, n, n, F, NI, NI, NI).transpose(3, 0, 4, 1, 5, 2, 6)
    return np.ascontiguousarray(g.reshape(F, n * NI, n * NI, n * NI))


def lattice_to_subgrids(U: np.ndarray) -> np.ndarray:
    F, N = U.shape[0], U.shape[1]
    n = N // NI
    g = U.reshape(F, n, NI, n, NI, n, NI).transpose(1, 3, 5, 0, 2, 4, 6)
    return np.ascontiguousarray(g.reshape(n ** 3, F, NI, NI, NI))


def initial_state(max_level: int, gamma: float = 5.0 / 3.0, omega: float = 0.3):
    I, dx = ho.rotating_star(8 ** max_level, gamma, omega)
    return subgrids_to_lattice(I), dx


def rhs(U: np.ndarray, max_level: int, gamma: float):
    N = U.shape[1]
    dx = 1.0 / N
    du, amax = ho.hydro_flux(ho.with_ghosts(lattice_to_subgrids(U)), dx, gamma)
    du = subgrids_to_lattice(du)
    g = fo.solve(U[0], max_level)[1:]
    L = du.copy()
    L[1] = du[1] + U[0] * g[0]
    L[2] = du[2] + U[0] * g[1]
    L[3] = du[3] + U[0] * g[2]
    L[4] = du[4] + ((U[1] * g[0] + U[2] * g[1]) + U[3] * g[2])
    return L, amax


def step(U: np.ndarray, max_level: int, gamma: float = 5.0 / 3.0, cfl: float = 0.4):
    """One SSP-RK2 step -> (U', dt)."""
    dx = 1.0 / U.shape[1]
    L1, amax = rhs(U, max_level, gamma)
    dt = (cfl * dx) / amax.max()
    U1 = U + dt * L1
    L2, _ = rhs(U1, max_level, gamma)
    return 0.5 * (U + (U1 + dt * L2)), dt


# ----------------------------------------------- sampled (full-size) checks --
# At max_level 3-5 the full oracle step is too slow for a test, but one stage
# of the step at a few sub-grids needs only those sub-grids' ghosted blocks
# (hydro) and gravity at their cells (the FMM oracle expands only the
# targets' ancestors). tests/test_gpu_star.py feeds these the GPU's own state
# before each stage, so every stage of every step is checked on the samples.
def ghosted_blocks(U: np.ndarray, subs: np.ndarray) -> np.ndarray:
    """[k, 5, 12, 12, 12] ghosted blocks (periodic) of sub-grids ``subs`` of
    the lattice U [5, N, N, N] (sub-grid s = (bz*n + by)*n + bx)."""
    N = U.shape[1]
    n = N // NI
    out = np.empty((len(subs), NF, NI + 4, NI + 4, NI + 4))
    for k, s in enumerate(subs):
        bz, by, bx = s // (n * n), (s // n) % n, s % n
        iz = (np.arange(-2, NI + 2) + NI * bz) % N
        iy = (np.arange(-2, NI + 2) + NI * by) % N
        ix = (np.arange(-2, NI + 2) + NI * bx) % N
        out[k] = U[:, iz][:, :, iy][:, :, :, ix]
    return out


def blocks(U: np.ndarray, subs: np.ndarray) -> np.ndarray:
    """[k, 5, 8, 8, 8] interiors of sub-grids ``subs``."""
    return ghosted_blocks(U, subs)[:, :, 2:-2, 2:-2, 2:-2]


def sub_targets(N: int, subs: np.ndarray) -> np.ndarray:
    """Leaf indices (x, y, z) [3, k*512] of the cells of ``subs``, in
    [k][z][y][x] order."""
    n = N // NI
    z, y, x = np.meshgrid(np.arange(NI), np.arange(NI), np.arange(NI), indexing="ij")
    t = []
    for s in subs:
        bz, by, bx = s // (n * n), (s // n) % n, s % n
        t.append(np.stack([x + NI * bx, y + NI * by, z + NI * bz]).reshape(3, -1))
    return np.concatenate(t, axis=1)


def sampled_rhs(U: np.ndarray, max_level: int, subs: np.ndarray, gamma: float = 5.0 / 3.0):
    """L(U) at the cells of sub-grids ``subs`` -> ([k, 5, 8, 8, 8], amax [k],
    g [3, k, 8, 8, 8]) — rhs() restricted to the samples."""
    N = U.shape[1]
    du, amax = ho.hydro_flux(ghosted_blocks(U, subs), 1.0 / N, gamma)
    g = fo.solve(U[0], max_level, sub_targets(N, subs))[1:]
    g = g.reshape(3, len(subs), NI, NI, NI)
    u = blocks(U, subs)
    L = du.copy()
    for c in range(3):
        L[:, 1 + c] = du[:, 1 + c] + u[:, 0] * g[c]
    L[:, 4] = du[:, 4] + ((u[:, 1] * g[0] + u[:, 2] * g[1]) + u[:, 3] * g[2])
    return L, amax, g
