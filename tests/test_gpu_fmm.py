"""K7 FMM gravity on the GPU against the self-authored oracle (PARITY
UNPINNED against the reference, which has no gravity). Tolerance — the
north_star's FP64 bar: per cell |dphi| <= 1e-10 |phi| and
|dg| <= 1e-10 |phi| / h (|phi|/h bounds the force's magnitude sum)."""

import math

import numpy as np
import pytest

from oracle import fmm_oracle as f

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL = 1e-10


def check(got, want, h):
    phi = np.abs(want[0])
    assert np.all(np.abs(got[0] - want[0]) <= TOL * phi), np.abs(got[0] / want[0] - 1).max()
    err = np.abs(got[1:] - want[1:]).max(axis=0)
    assert np.all(err <= TOL * phi / h), (err / (phi / h)).max()


def solver(L):
    from paper_2303_08058_b200.gravity import GravitySolver
    return GravitySolver(L, torch.device("cuda", 0))


@pytest.mark.parametrize("L,seed", [(1, None), (1, 5), (2, None)])
def test_fmm_full_lattice_vs_oracle(L, seed):
    rho = f.rotating_star_density(L)
    if seed is not None:
        rho = rho * (1 + 0.3 * np.random.default_rng(seed).random(rho.shape))
    s = solver(L)
    got = s.solve(torch.from_numpy(rho).cuda()).cpu().numpy()
    if L == 1:
        want = f.solve(rho, L)
        check(got, want, 1 / rho.shape[0])
    else:
        N = rho.shape[0]
        tg = np.random.default_rng(7).integers(0, N, size=(3, 400))
        tg = np.concatenate([tg, np.array([[0, 0, 0], [N - 1] * 3, [0, N - 1, 3]]).T], axis=1)
        check(got[:, tg[2], tg[1], tg[0]], f.solve(rho, L, tg), 1 / N)


def test_fmm_upward_moments_vs_oracle():
    L = 2
    rho = np.random.default_rng(11).random((32, 32, 32)) + 0.05
    s = solver(L)
    s.upward(torch.from_numpy(rho).cuda())
    torch.cuda.synchronize()
    work = s.work.cpu().numpy()
    Ms = f.upward(rho, L)
    scale = np.array([(1.0 if len(B) % 2 else -1.0) * f.mult(B) / math.factorial(len(B))
                      for B in f.COMPS])
    import ctypes
    from paper_2303_08058_b200 import _native as N
    info = (ctypes.c_uint64 * 8)()
    for lev in range(L):
        N.call("tb_fmm_slab_layout", L, 1, 0, lev, info)
        raw_off, red_off, n, halo = info[0] // 8, info[1] // 8, info[3], info[6]
        cells = n ** 3
        got = np.moveaxis(work[raw_off:raw_off + 20 * cells].reshape((n,) * 3 + (20,)), -1, 0)
        want = Ms[lev] * scale[:, None, None, None]
        mag = np.abs(want).max(axis=(1, 2, 3), keepdims=True)
        assert np.all(np.abs(got - want) <= 1e-13 * mag + 1e-300), lev
        recs = work[red_off:red_off + 18 * n * n * (n + 2 * halo)].reshape(-1, 18)
        assert np.all(recs[:n * n * halo] == 0.0) and np.all(recs[n * n * (n + halo):] == 0.0)
        red = recs[n * n * halo:n * n * (n + halo)]
        w = want.reshape(20, cells)
        # traceless reduction: zz-containing moments folded into xx, yy, xxx, ...
        exp = np.stack([w[0], w[1], w[2], w[3], w[4] - w[9], w[5], w[6], w[7] - w[9], w[8],
                        w[10] - w[15], w[11] - w[18], w[12] - w[19], w[13] - w[15], w[14],
                        w[16] - w[18], w[17] - w[19]], axis=1)
        assert np.all(np.abs(red[:, :16] - exp) <= 1e-13 * np.abs(w).max() + 1e-300), lev
        assert np.all(red[:, 16:] == 0.0)


@pytest.mark.parametrize("L", [3, 4])
def test_fmm_at_config3_size_sampled(L):
    """BASELINE config 3 (max_level 4): sampled cells vs the oracle's subset
    solve (which expands only the samples' ancestors)."""
    rho = f.rotating_star_density(L)
    N = rho.shape[0]
    s = solver(L)
    got = s.solve(torch.from_numpy(rho).cuda()).cpu().numpy()
    tg = np.random.default_rng(L).integers(0, N, size=(3, 96))
    tg = np.concatenate([tg, np.array([[0, 0, 0], [N - 1] * 3, [N // 2] * 3]).T], axis=1)
    check(got[:, tg[2], tg[1], tg[0]], f.solve(rho, L, tg), 1 / N)
    assert np.isfinite(got).all()


def test_fmm_mirror_symmetry_and_repeatability():
    L = 3
    rho = torch.from_numpy(f.rotating_star_density(L)).cuda()
    s = solver(L)
    a = s.solve(rho).clone()
    b = s.solve(rho).clone()
    assert torch.equal(a, b)                      # deterministic (no atomics)
    fl = torch.flip(a, dims=[3])
    assert torch.allclose(a[0], fl[0], rtol=1e-12, atol=0)
    assert torch.allclose(a[1], -fl[1], rtol=0, atol=1e-9 * a[1].abs().max().item())


def test_fmm_rejects_bad_input():
    s = solver(1)
    with pytest.raises(ValueError):
        s.solve(torch.zeros((8, 8, 8), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        s.solve(torch.zeros((16, 16, 16), dtype=torch.float32, device="cuda"))
