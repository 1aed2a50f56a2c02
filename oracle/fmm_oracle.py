"""numpy oracle for the FMM gravity kernels (K7) — TEST INFRASTRUCTURE.

PARITY UNPINNED: the reference contains no gravity solver (SURVEY.md §0:
SPEC.md:17,490 put "FMM gravity solver, §2.1" out of scope; PAPER.md:247-259
only cites Octo-Tiger's FMM). The north_star names "the FMM monopole/
multipole stencil-interaction kernels" (BASELINE.json config 3: "FMM
multipole+monopole interaction kernels only, rotating star max_level 4"), so
this module is a SELF-AUTHORED specification in the spirit of Octo-Tiger's
Cartesian FMM (order-3 multipoles, an opening-angle stencil at every level of
the octree, monopoles at the leaves). What is pinned:

1. GPU vs this restatement per cell, within the north_star's FP64 tolerance
   (relative error <= 1e-10 on the potential, force error <= 1e-10 * |phi|/h —
   each force term m/r^2 is bounded by (m/r)/h, so |phi|/h bounds the force's
   magnitude sum and the tolerance is relative to it);
2. properties of the spec itself: every ordered leaf pair is covered exactly
   once by the interaction lists (tests/test_fmm_oracle.py), the result
   converges to the direct O(N^2) sum (order-3 truncation, theta = 1/2), and
   mirror symmetry of a symmetric mass distribution.

Spec
----
* Uniform octree of depth ``L`` (max_level) over the cube [-1/2, 1/2)^3: level
  ``l`` holds 8^l sub-grids of 8^3 cells, i.e. a lattice of N_l = 8 * 2^l cells
  per edge with cell size h_l = 1/N_l and centres (i + 1/2) h_l - 1/2. Cell i at
  level l has parent i >> 1 (per axis) at level l-1. Outside the cube there is
  no mass (isolated boundary).
* Arrays are global lattices [.., N, N, N] (z, y, x; x fastest).
* Leaves (level L) are monopoles: m = rho * h_L^3 at the cell centre.
* Multipoles: raw Cartesian moments about the geometric cell centre X,
  M^(n)_{a..} = sum_k m_k (x_k - X)_a ..., n <= 3, symmetric storage in the
  20-component order COMPS below. Parent moments come from the 8 children by
  the exact shift (M2M) of raw moments.
* theta = 1/2: two cells of one level are "near" iff their integer offset o
  has |o|^2 <= (1/theta)^2 = 4. Parent-near offsets: PNEAR (33 entries).
* Level l in [1, L-1] (multipole interactions, M2L): target i receives from
  every j = 2((i >> 1) + P) + c, P in PNEAR, c in {0,1}^3, with |j - i|^2 > 4.
  Level 0: from every j of the 8^3 lattice with |j - i|^2 > 4.
  With R = X_i - X_j and D^(n) the n-th derivative tensor of 1/r at R:
      L^(n)_A += -sum_{m <= 3-n} ((-1)^m / m!) sum_B mult(B) M^(m)_B D^(n+m)_{A+B}
  so phi(X_i + y) = sum_n L^(n) . y^n / n!  (phi = -sum m/r, G = 1).
* Downward (L2L): a child at X_c = X_p + d adds
      L^(n)_A(child) += sum_{k <= 3-n} (1/k!) sum_B mult(B) L^(n+k)_{A+B}(parent) d^B.
* Leaves (monopole interactions, P2P): target i sums -m_j/r and the gradient
  m_j R/r^3 over every j = 2((i >> 1) + P) + c (P in PNEAR, c in {0,1}^3),
  j != i; plus the parent's (level L-1) expansion evaluated at the leaf centre
  (L2P). Output per leaf: phi and g = -grad phi, as [4, N, N, N]
  (phi, gx, gy, gz).
Every ordered pair of distinct leaves is then accounted for exactly once.
"""

from __future__ import annotations

from math import factorial
from typing import Dict, List, Tuple

import numpy as np

COMPS: List[Tuple[int, ...]] = [
    (),
    (0,), (1,), (2,),
    (0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2),
    (0, 0, 0), (0, 0, 1), (0, 0, 2), (0, 1, 1), (0, 1, 2), (0, 2, 2),
    (1, 1, 1), (1, 1, 2), (1, 2, 2), (2, 2, 2),
]
NC = len(COMPS)                      # 20
INDEX: Dict[Tuple[int, ...], int] = {t: k for k, t in enumerate(COMPS)}
ORDER = [len(t) for t in COMPS]
THETA_NEAR2 = 4                      # (1/theta)^2, theta = 1/2


def mult(t: Tuple[int, ...]) -> int:
    """Number of index tuples that sort to ``t``."""
    out = factorial(len(t))
    for a in range(3):
        out //= factorial(t.count(a))
    return out


PNEAR = [(px, py, pz) for pz in range(-2, 3) for py in range(-2, 3) for px in range(-2, 3)
         if px * px + py * py + pz * pz <= THETA_NEAR2]          # 33 offsets, (x, y, z)
CHILD = [(cx, cy, cz) for cz in (0, 1) for cy in (0, 1) for cx in (0, 1)]


def m2l_terms():
    """(target comp, source comp, D comp, coefficient) of the M2L contraction."""
    terms = []
    for t, A in enumerate(COMPS):
        for s, B in enumerate(COMPS):
            m = len(B)
            if len(A) + m > 3:
                continue
            coef = -((-1) ** m) / factorial(m) * mult(B)
            terms.append((t, s, INDEX[tuple(sorted(A + B))], coef))
    return terms


def l2l_terms():
    """(child comp, parent comp, monomial comp of d, coefficient)."""
    terms = []
    for t, A in enumerate(COMPS):
        for b, B in enumerate(COMPS):
            k = len(B)
            if len(A) + k > 3:
                continue
            terms.append((t, INDEX[tuple(sorted(A + B))], b, mult(B) / factorial(k)))
    return terms


def m2m_terms():
    """(parent comp, child comp, monomial comp of d, integer coefficient):
    prod_a (s_a + d_a) expanded over subsets of the index positions."""
    acc: Dict[Tuple[int, int, int], int] = {}
    for t, A in enumerate(COMPS):
        n = len(A)
        for mask in range(1 << n):
            S = tuple(sorted(A[q] for q in range(n) if mask >> q & 1))       # -> d
            rest = tuple(sorted(A[q] for q in range(n) if not mask >> q & 1))  # -> s
            key = (t, INDEX[rest], INDEX[S])
            acc[key] = acc.get(key, 0) + 1
    return [(t, s, b, c) for (t, s, b), c in sorted(acc.items())]


M2L_TERMS = m2l_terms()
L2L_TERMS = l2l_terms()
M2M_TERMS = m2m_terms()


def monomials(d: np.ndarray) -> np.ndarray:
    """d^B for every comp B: d [3, ...] -> [20, ...]."""
    out = np.empty((NC,) + d.shape[1:])
    for k, B in enumerate(COMPS):
        v = np.ones(d.shape[1:])
        for a in B:
            v = v * d[a]
        out[k] = v
    return out


def d_tensor(R: np.ndarray) -> np.ndarray:
    """Derivatives of 1/r at R ([3, ...]) up to order 3 -> [20, ...]."""
    r2 = (R[0] * R[0] + R[1] * R[1]) + R[2] * R[2]
    r1 = 1.0 / np.sqrt(r2)
    i2 = r1 * r1
    r3 = r1 * i2
    r5 = r3 * i2
    r7 = r5 * i2
    D = np.empty((NC,) + R.shape[1:])
    for k, A in enumerate(COMPS):
        n = len(A)
        if n == 0:
            D[k] = r1
        elif n == 1:
            D[k] = -R[A[0]] * r3
        elif n == 2:
            a, b = A
            D[k] = 3.0 * R[a] * R[b] * r5 - (r3 if a == b else 0.0)
        else:
            a, b, c = A
            v = -15.0 * R[a] * R[b] * R[c] * r7
            t = (R[a] if b == c else 0.0) + (R[b] if a == c else 0.0) + (R[c] if a == b else 0.0)
            D[k] = v + 3.0 * r5 * t
    return D


def lattice(level: int) -> int:
    return 8 << level


def centres(level: int, idx: np.ndarray) -> np.ndarray:
    """Centres of integer cells idx [3, ...] (x, y, z) at ``level``."""
    h = 1.0 / lattice(level)
    return (idx + 0.5) * h - 0.5


# ------------------------------------------------------------ upward pass --
def leaf_moments(rho: np.ndarray) -> np.ndarray:
    """[N,N,N] density -> [1, N, N, N] leaf multipoles: monopoles only (every
    higher leaf moment is zero about the cell centre, so only the monopole
    component is stored — max_level 5 would otherwise need 2.7 GB)."""
    N = rho.shape[0]
    h = 1.0 / N
    return (rho * (h * h * h))[None]


def m2m(Mc: np.ndarray) -> np.ndarray:
    """Children moments [20 or 1, 2N, 2N, 2N] -> parent moments [20, N, N, N]."""
    n2 = Mc.shape[1]
    hc = 1.0 / n2
    Mp = np.zeros((NC, n2 // 2, n2 // 2, n2 // 2))
    for cx, cy, cz in CHILD:
        # child centre - parent centre = (c - 1/2) * h_child per axis
        d = np.array([(cx - 0.5) * hc, (cy - 0.5) * hc, (cz - 0.5) * hc])
        mono = monomials(d.reshape(3, 1))[:, 0]
        sub = Mc[:, cz::2, cy::2, cx::2]
        for t, s, b, c in M2M_TERMS:
            if s < sub.shape[0]:           # a monopole-only child level
                Mp[t] += (c * mono[b]) * sub[s]
    return Mp


def upward(rho: np.ndarray, max_level: int) -> List[np.ndarray]:
    """Moments of every level 0..max_level (index = level)."""
    Ms = [None] * (max_level + 1)
    Ms[max_level] = leaf_moments(rho)
    for lev in range(max_level - 1, -1, -1):
        Ms[lev] = m2m(Ms[lev + 1])
    return Ms


# ------------------------------------------------------ interaction lists --
def _grid_idx(N: int) -> np.ndarray:
    z, y, x = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    return np.stack([x, y, z]).reshape(3, -1)             # (x, y, z) of flat cells


def partner_offsets(level: int, targets: np.ndarray):
    """Yield (j [3, n], mask [n]) over the stencil of ``targets`` [3, n]:
    the M2L interaction list at ``level`` (j in range, |j - i|^2 > 4)."""
    N = lattice(level)
    if level == 0:
        for j in _grid_idx(N).T:
            jj = np.broadcast_to(j[:, None], targets.shape)
            o = jj - targets
            yield jj, (o * o).sum(0) > THETA_NEAR2
        return
    par = targets >> 1
    for P in PNEAR:
        for c in CHILD:
            j = 2 * (par + np.array(P)[:, None]) + np.array(c)[:, None]
            o = j - targets
            ok = ((j >= 0) & (j < N)).all(0) & ((o * o).sum(0) > THETA_NEAR2)
            yield j, ok


def _gather(A: np.ndarray, j: np.ndarray, ok: np.ndarray) -> np.ndarray:
    """A [C, N, N, N] at cells j [3, n] (zeros where not ok)."""
    N = A.shape[1]
    jc = np.clip(j, 0, N - 1)
    out = A[:, jc[2], jc[1], jc[0]]
    return np.where(ok[None, :], out, 0.0)


# ------------------------------------------------------------ interactions --
def m2l(M: np.ndarray, level: int, targets: np.ndarray) -> np.ndarray:
    """Local expansions [20, n] of ``targets`` [3, n] from level-``level``
    multipoles M [20, N, N, N] over the interaction list."""
    L = np.zeros((NC, targets.shape[1]))
    Xi = centres(level, targets)
    for j, ok in partner_offsets(level, targets):
        if not ok.any():
            continue
        R = Xi - centres(level, j)
        R = np.where(ok[None, :], R, 1.0)                  # avoid r = 0 off-list
        D = d_tensor(R)
        Ms = _gather(M, j, ok)
        for t, s, d, c in M2L_TERMS:
            L[t] += c * Ms[s] * D[d]
    return L


def l2l(Lp: np.ndarray, d: np.ndarray) -> np.ndarray:
    """Shift parent expansions Lp [20, n] by d [3, n] (child - parent centre)."""
    mono = monomials(d)
    Lc = np.zeros_like(Lp)
    for t, p, b, c in L2L_TERMS:
        Lc[t] += c * Lp[p] * mono[b]
    return Lc


def p2p(rho: np.ndarray, targets: np.ndarray) -> np.ndarray:
    """Leaf monopole interactions -> [4, n] (phi, dphi/dx, dphi/dy, dphi/dz)."""
    N = rho.shape[0]
    h = 1.0 / N
    out = np.zeros((4, targets.shape[1]))
    Xi = (targets + 0.5) * h - 0.5
    m = rho[None] * (h * h * h)
    for j, ok in leaf_partners(N, targets):
        R = Xi - ((j + 0.5) * h - 0.5)
        R = np.where(ok[None, :], R, 1.0)
        mj = _gather(m, j, ok)[0]
        r2 = (R[0] * R[0] + R[1] * R[1]) + R[2] * R[2]
        r1 = 1.0 / np.sqrt(r2)
        mr = mj * r1
        mr3 = mr * (r1 * r1)
        out[0] -= mr
        out[1] += mr3 * R[0]
        out[2] += mr3 * R[1]
        out[3] += mr3 * R[2]
    return out


def leaf_partners(N: int, targets: np.ndarray):
    """Yield (j [3, n], mask [n]) over the leaf (P2P) stencil of ``targets``
    on an N^3 leaf lattice: every child of a parent-near parent, j != i, in
    range."""
    par = targets >> 1
    for P in PNEAR:
        for c in CHILD:
            j = 2 * (par + np.array(P)[:, None]) + np.array(c)[:, None]
            ok = ((j >= 0) & (j < N)).all(0) & (j != targets).any(0)
            yield j, ok


def solve(rho: np.ndarray, max_level: int, targets: np.ndarray | None = None):
    """Gravity of the leaves: [4, n] = (phi, gx, gy, gz) at ``targets``
    ([3, n] leaf indices, default: every leaf, returned as [4, N, N, N]).

    Only the ancestors of the targets are expanded, so a handful of targets
    at max_level 4-5 costs seconds (full-size spot checks)."""
    N = lattice(max_level)
    assert rho.shape == (N, N, N)
    full = targets is None
    if full:
        targets = _grid_idx(N)
    Ms = upward(rho, max_level)
    # ancestors' local expansions, root to parent of the leaves
    Lacc = None
    for lev in range(0, max_level):
        anc = targets >> (max_level - lev)
        # each distinct ancestor once (many targets share one), then scatter
        uniq, inv = np.unique(anc, axis=1, return_inverse=True)
        Ll = m2l(Ms[lev], lev, uniq)[:, inv.reshape(-1)]
        if Lacc is not None:
            # child centre - parent centre, per target's ancestor at lev
            hc = 1.0 / lattice(lev)
            d = ((anc & 1) - 0.5) * hc
            Ll = Ll + l2l(Lacc, d)
        Lacc = Ll
    out = p2p(rho, targets)
    if Lacc is not None:
        h = 1.0 / N
        d = ((targets & 1) - 0.5) * h                      # leaf - parent centre
        mono = monomials(d)
        phi = np.zeros(targets.shape[1])
        grad = np.zeros((3, targets.shape[1]))
        for t, p, b, c in L2L_TERMS:
            if t == 0:
                phi += c * Lacc[p] * mono[b]
            elif t <= 3:
                grad[t - 1] += c * Lacc[p] * mono[b]
        out[0] += phi
        out[1:] += grad
    out[1:] = -out[1:]
    if full:
        return out.reshape(4, N, N, N)
    return out


def direct(rho: np.ndarray, targets: np.ndarray, chunk: int = 512) -> np.ndarray:
    """Exact O(N^2) gravity of all leaf monopoles at ``targets`` -> [4, n]."""
    N = rho.shape[0]
    h = 1.0 / N
    src = _grid_idx(N)
    m = (rho.reshape(-1) * (h * h * h))
    nz = m != 0.0
    src, m = src[:, nz], m[nz]
    Xs = (src + 0.5) * h - 0.5
    Xt = (targets + 0.5) * h - 0.5
    out = np.zeros((4, targets.shape[1]))
    for a in range(0, targets.shape[1], chunk):
        R = Xt[:, a:a + chunk, None] - Xs[:, None, :]
        r2 = (R * R).sum(0)
        same = r2 == 0.0
        r2 = np.where(same, 1.0, r2)
        r1 = np.where(same, 0.0, 1.0 / np.sqrt(r2))
        mr = m[None, :] * r1
        out[0, a:a + chunk] = -mr.sum(1)
        mr3 = mr * r1 * r1
        for k in range(3):
            out[1 + k, a:a + chunk] = -(mr3 * R[k]).sum(1)
    return out


# ------------------------------------------------------- synthetic inputs --
def rotating_star_density(max_level: int) -> np.ndarray:
    """The hydro oracle's synthetic rotating star (a polytrope-like bump on a
    low floor, oracle/hydro_oracle.py:rotating_star) as a [N, N, N] density
    lattice at ``max_level`` (N = 8 * 2^L), on the isolated unit cube."""
    N = lattice(max_level)
    c = (np.arange(N) + 0.5) / N - 0.5
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    r = np.sqrt(x * x + y * y + z * z)
    return 1e-3 + np.clip(1.0 - (r / 0.35) ** 2, 0.0, None) ** 1.5
