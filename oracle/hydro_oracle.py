"""numpy oracle for the hydro reconstruct-and-flux kernel — TEST INFRASTRUCTURE.

PARITY UNPINNED: the reference contains no hydro code (SURVEY.md §0:
SPEC.md:17,490; src/miniapp.py:12-13 — "the arithmetic is deliberately
trivial"). The north_star names Octo-Tiger's hydro reconstruct+flux kernels
(PAPER.md:247-259 cites, but does not specify, them), so this module is a
SELF-AUTHORED specification of such a kernel, restated exactly by the CUDA
kernel (tb_hydro_flux). What is pinned is (1) bit-identity between this
restatement and the GPU and (2) physics properties that hold whatever the
reference would have been: exact zero update of uniform states,
mirror-symmetry, and conservation of mass/momentum/energy to round-off over a
periodic lattice of sub-grids.

Spec (one batch of sub-grids, each 8^3 interior cells with a 2-cell ghost
layer, i.e. 12^3 cells):

* layout U[s, f, k, j, i], f in (rho, sx, sy, sz, E), i fastest, float64;
* ideal gas, gamma given; primitives per cell, in this exact order:
  irho = 1/rho; vx = sx*irho; vy = sy*irho; vz = sz*irho;
  ke = 0.5 * ((sx*vx + sy*vy) + sz*vz); p = (gamma - 1) * (E - ke);
  (one divide per cell; the reciprocals 1/(gamma-1) and 1/dx are formed once)
* piecewise-linear reconstruction of (rho, vx, vy, vz, p) along each
  direction with the minmod limiter: dl = q[c]-q[c-1], dr = q[c+1]-q[c];
  slope = 0 if dl*dr <= 0 else (dl if |dl| < |dr| else dr);
  face values q[c] +/- 0.5*slope;
* at each face: left state = cell c's "+" value, right state = cell c+1's "-"
  value; per state (direction d with normal velocity vn):
  cs = sqrt((gamma*p)/rho); e = p*(1/(gamma-1)) + 0.5*rho*((vx*vx + vy*vy) + vz*vz);
  U = (rho, rho*vx, rho*vy, rho*vz, e); F = (rho*vn, rho*vx*vn [+p if d==x],
  rho*vy*vn [+p if d==y], rho*vz*vn [+p if d==z], (e+p)*vn) with momentum
  flux components computed as (rho*v_comp)*vn then + p on the normal one;
* Kurganov-Tadmor / local Lax-Friedrichs flux (the central scheme family
  Octo-Tiger's hydro uses): a = max(|vnL| + csL, |vnR| + csR);
  F = 0.5*(FL + FR) - 0.5*a*(UR - UL), computed as
  (0.5*(FL+FR)) - ((0.5*a)*(UR-UL));
* update of interior cell c: du = (Fx[c+1/2]-Fx[c-1/2]);
  du = du + (Fy[c+1/2]-Fy[c-1/2]); du = du + (Fz[c+1/2]-Fz[c-1/2]);
  dUdt = -(du * (1/dx));
* per sub-grid: amax = max over all its faces of a (the CFL signal speed).
"""

from __future__ import annotations

import numpy as np

NG = 2                      # ghost width
NI = 8                      # interior cells per edge
NT = NI + 2 * NG            # 12 cells per edge with ghosts
NF = 5                      # rho, sx, sy, sz, E


def primitives(U: np.ndarray, gamma: float):
    rho, sx, sy, sz, E = (U[:, f] for f in range(NF))
    irho = 1.0 / rho
    vx = sx * irho
    vy = sy * irho
    vz = sz * irho
    ke = 0.5 * ((sx * vx + sy * vy) + sz * vz)
    p = (gamma - 1.0) * (E - ke)
    return rho, vx, vy, vz, p


def _minmod(dl, dr):
    pick = np.where(np.abs(dl) < np.abs(dr), dl, dr)
    return np.where(dl * dr <= 0.0, 0.0, pick)


def _state(rho, vx, vy, vz, p, gamma, d):
    cs = np.sqrt((gamma * p) / rho)
    e = p * (1.0 / (gamma - 1.0)) + 0.5 * rho * ((vx * vx + vy * vy) + vz * vz)
    vn = (vx, vy, vz)[d]
    mx, my, mz = rho * vx, rho * vy, rho * vz
    U = (rho, mx, my, mz, e)
    fmx, fmy, fmz = mx * vn, my * vn, mz * vn
    if d == 0:
        fmx = fmx + p
    elif d == 1:
        fmy = fmy + p
    else:
        fmz = fmz + p
    F = (rho * vn, fmx, fmy, fmz, (e + p) * vn)
    return U, F, np.abs(vn) + cs


def face_fluxes(W, gamma, d):
    """Fluxes through the faces between cells c and c+1 along axis d
    (array axis 3-d of [s, k, j, i]), for c = 1 .. 9 (faces 1.5 .. 9.5),
    restricted to interior transverse cells. Returns (F[5] arrays, a)."""
    axis = 3 - d                           # i -> axis 3, j -> 2, k -> 1
    q = [w for w in W]                     # rho, vx, vy, vz, p

    def sl(a, lo, hi):
        idx = [slice(None)] * 4
        idx[axis] = slice(lo, hi)
        for ax in range(1, 4):
            if ax != axis:
                idx[ax] = slice(NG, NG + NI)
        return a[tuple(idx)]

    # cells c-1, c, c+1, c+2 for c = 1..9  ->  index ranges
    L, R = [], []
    for v in q:
        qm, q0, qp, qpp = sl(v, 0, 9), sl(v, 1, 10), sl(v, 2, 11), sl(v, 3, 12)
        s0 = _minmod(q0 - qm, qp - q0)          # slope at c
        s1 = _minmod(qp - q0, qpp - qp)         # slope at c+1
        L.append(q0 + 0.5 * s0)
        R.append(qp - 0.5 * s1)
    UL, FL, aL = _state(*L, gamma, d)
    UR, FR, aR = _state(*R, gamma, d)
    a = np.maximum(aL, aR)
    F = [(0.5 * (fl + fr)) - ((0.5 * a) * (ur - ul))
         for fl, fr, ul, ur in zip(FL, FR, UL, UR)]
    return F, a


def hydro_flux(U: np.ndarray, dx: float, gamma: float):
    """dU/dt for the interior cells ([s, 5, 8, 8, 8]) and amax per sub-grid."""
    assert U.ndim == 5 and U.shape[1:] == (NF, NT, NT, NT)
    W = primitives(U, gamma)
    s = U.shape[0]
    du = None
    amax = np.full(s, -np.inf)
    for d in range(3):
        F, a = face_fluxes(W, gamma, d)
        axis = 3 - d
        amax = np.maximum(amax, a.reshape(s, -1).max(axis=1))
        parts = []
        for f in range(NF):
            lo = np.take(F[f], np.arange(0, NI), axis=axis)     # face c-1/2
            hi = np.take(F[f], np.arange(1, NI + 1), axis=axis)  # face c+1/2
            parts.append(hi - lo)
        diff = np.stack(parts, axis=1)
        du = diff if du is None else du + diff
    return -(du * (1.0 / dx)), amax


# ------------------------------------------------------- synthetic inputs --
def lattice_shape(subgrids: int):
    n = round(subgrids ** (1.0 / 3.0))
    if n ** 3 != subgrids:
        raise ValueError("subgrids must be a cube (a uniform octree level)")
    return n


def rotating_star(subgrids: int, gamma: float = 5.0 / 3.0, omega: float = 0.3):
    """Synthetic 'rotating star' on a periodic lattice of n^3 sub-grids in the
    unit cube: a smooth polytrope-like density bump in solid-body rotation
    about z, on a low ambient floor. Returns the interior conserved state
    [n^3, 5, 8, 8, 8] (sub-grid order: x fastest) and dx."""
    n = lattice_shape(subgrids)
    N = n * NI
    dx = 1.0 / N
    c = (np.arange(N) + 0.5) * dx - 0.5
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    r = np.sqrt(x * x + y * y + z * z)
    rho = 1e-3 + np.clip(1.0 - (r / 0.35) ** 2, 0.0, None) ** 1.5
    vx, vy, vz = -omega * y, omega * x, np.zeros_like(x)
    p = 1e-4 + 0.3 * rho ** gamma
    E = p / (gamma - 1.0) + 0.5 * rho * (vx * vx + vy * vy + vz * vz)
    glob = np.stack([rho, rho * vx, rho * vy, rho * vz, E])      # [5, N, N, N]
    g = glob.reshape(NF, n, NI, n, NI, n, NI).transpose(1, 3, 5, 0, 2, 4, 6)
    return np.ascontiguousarray(g.reshape(subgrids, NF, NI, NI, NI)), dx


def with_ghosts(interior: np.ndarray):
    """Fill 2-cell ghost layers from the periodic lattice neighbours (this is
    what the octree's ghost exchange provides) -> [s, 5, 12, 12, 12]."""
    s = interior.shape[0]
    n = lattice_shape(s)
    N = n * NI
    glob = interior.reshape(n, n, n, NF, NI, NI, NI).transpose(3, 0, 4, 1, 5, 2, 6)
    glob = glob.reshape(NF, N, N, N)
    pad = np.pad(glob, ((0, 0), (NG, NG), (NG, NG), (NG, NG)), mode="wrap")
    out = np.empty((s, NF, NT, NT, NT))
    for bz in range(n):
        for by in range(n):
            for bx in range(n):
                out[(bz * n + by) * n + bx] = pad[:, bz * NI:bz * NI + NT,
                                                  by * NI:by * NI + NT,
                                                  bx * NI:bx * NI + NT]
    return out


def euler_step(I: np.ndarray, gamma: float = 5.0 / 3.0, cfl: float = 0.4):
    """One forward-Euler hydro step of the periodic sub-grid lattice (the
    native machine's hydro workload, tb_machine_run_hydro): dt =
    (cfl * dx) / max(amax); I' = I + dt * dU/dt. Returns (I', dt)."""
    n = lattice_shape(I.shape[0])
    dx = 1.0 / (n * NI)
    du, amax = hydro_flux(with_ghosts(I), dx, gamma)
    dt = (cfl * dx) / amax.max()
    return I + dt * du, dt
