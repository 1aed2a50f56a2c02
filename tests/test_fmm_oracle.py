"""Self-authored FMM oracle (PARITY UNPINNED — the reference has no gravity):
properties of the spec itself, checked on CPU."""

import numpy as np
import pytest

from oracle import fmm_oracle as f


def test_tables():
    assert len(f.PNEAR) == 33
    assert len(f.M2L_TERMS) == len(f.L2L_TERMS) == len(f.M2M_TERMS) == 84
    assert sum(f.mult(t) for t in f.COMPS if len(t) == 3) == 27


@pytest.mark.parametrize("L", [1, 2])
def test_every_leaf_pair_is_covered_exactly_once(L):
    """P2P partners at the leaves plus the descendants of the M2L partners of
    every ancestor cover each other leaf exactly once (and never the target)."""
    N = f.lattice(L)
    rng = np.random.default_rng(L)
    targets = np.concatenate([rng.integers(0, N, size=(3, 12)),
                              np.array([[0, 0, 0], [N - 1] * 3]).T], axis=1)
    for k in range(targets.shape[1]):
        i = targets[:, k:k + 1]
        cnt = np.zeros((N, N, N), dtype=np.int64)
        for j, ok in f.leaf_partners(N, i):
            if ok[0]:
                cnt[j[2, 0], j[1, 0], j[0, 0]] += 1
        for lev in range(L):
            anc = i >> (L - lev)
            s = 1 << (L - lev)
            for j, ok in f.partner_offsets(lev, anc):
                if ok[0]:
                    x, y, z = (j[:, 0] * s).tolist()
                    cnt[z:z + s, y:y + s, x:x + s] += 1
        want = np.ones_like(cnt)
        want[i[2, 0], i[1, 0], i[0, 0]] = 0
        assert np.array_equal(cnt, want)


def test_m2l_truncation_error_scales_as_order_three():
    """A cell's order-3 expansion: relative potential error ~ (a/R)^4."""
    rng = np.random.default_rng(1)
    ms = rng.random(8)
    pos = np.array([[c[0] - 0.5, c[1] - 0.5, c[2] - 0.5] for c in f.CHILD]).T
    M = np.array([np.prod([pos[a] for a in B], axis=0).dot(ms) if B else ms.sum()
                  for B in f.COMPS])
    errs = []
    for R in (4.0, 8.0, 16.0):
        X = np.array([R, 0.7 * R, 0.3 * R])
        D = f.d_tensor(X.reshape(3, 1))[:, 0]
        Lx = np.zeros(20)
        for t, s, d, c in f.M2L_TERMS:
            Lx[t] += c * M[s] * D[d]
        Rk = X[:, None] - pos
        exact = -(ms / np.sqrt((Rk * Rk).sum(0))).sum()
        errs.append(abs(Lx[0] - exact) / abs(exact))
    assert errs[0] / errs[1] > 12 and errs[1] / errs[2] > 12


def test_m2m_is_the_exact_moment_shift():
    rng = np.random.default_rng(2)
    rho = rng.random((16, 16, 16))
    Ms = f.upward(rho, 1)
    h = 1 / 16
    m = rho * h ** 3
    z, y, x = np.meshgrid(np.arange(16), np.arange(16), np.arange(16), indexing="ij")
    # parent (0,0,0) of level 0 covers leaves [0,2)^3; centre at (0.5*2 h) - 0.5
    sel = (x < 2) & (y < 2) & (z < 2)
    X = 1 * h - 0.5
    d = [(x[sel] + 0.5) * h - 0.5 - X, (y[sel] + 0.5) * h - 0.5 - X, (z[sel] + 0.5) * h - 0.5 - X]
    for k, B in enumerate(f.COMPS):
        v = m[sel].copy()
        for a in B:
            v = v * d[a]
        assert abs(Ms[0][k, 0, 0, 0] - v.sum()) <= 1e-15 * (abs(v).sum() + 1e-300)


@pytest.mark.parametrize("L", [1])
def test_fmm_converges_to_direct_sum(L):
    rho = f.rotating_star_density(L)
    out = f.solve(rho, L)
    N = rho.shape[0]
    rng = np.random.default_rng(3)
    tg = rng.integers(0, N, size=(3, 300))
    d = f.direct(rho, tg)
    got = out[:, tg[2], tg[1], tg[0]]
    assert np.abs((got[0] - d[0]) / d[0]).max() < 5e-4
    assert np.abs(got[1:] - d[1:]).max() < 5e-3 * np.abs(d[1:]).max()


def test_subset_solve_equals_full_solve():
    rho = np.random.default_rng(4).random((16, 16, 16)) + 0.1
    full = f.solve(rho, 1)
    tg = np.array([[0, 5, 15, 7], [0, 9, 15, 8], [0, 2, 15, 8]])
    sub = f.solve(rho, 1, tg)
    assert np.array_equal(sub, full[:, tg[2], tg[1], tg[0]])


def test_mirror_symmetry():
    rho = f.rotating_star_density(1)            # symmetric under x -> -x
    out = f.solve(rho, 1)
    flipped = out[:, :, :, ::-1]
    assert np.allclose(out[0], flipped[0], rtol=1e-12, atol=0)
    assert np.allclose(out[1], -flipped[1], rtol=1e-9, atol=1e-12 * np.abs(out[1]).max())
    assert np.allclose(out[2], flipped[2], rtol=1e-9, atol=1e-12 * np.abs(out[2]).max())


def test_product_density_matches_the_oracle_generator():
    pytest.importorskip("torch")
    from paper_2303_08058_b200.gravity import rotating_star_density
    for L in (1, 2):
        np.testing.assert_allclose(rotating_star_density(L).numpy(),
                                   f.rotating_star_density(L), rtol=1e-15, atol=0)
