"""The coupled rotating-star step on the GPU vs its self-authored oracle
(PARITY UNPINNED against the reference, which has no physics). Tolerance —
the north_star's FP64 bar: every cell's conserved variables within 1e-10
relative (momentum components relative to the cell's |s| + 1e-6 max|s|, as
they pass through zero), dt within 1e-12; mass conserved to round-off."""

import numpy as np
import pytest

from oracle import star_oracle as so

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def close(got, want):
    for f in range(5):
        w, g = want[f], got[f]
        scale = np.abs(w) + (1e-6 * np.abs(w).max() if f in (1, 2, 3) else 0.0)
        err = np.abs(g - w) / scale
        assert err.max() <= 1e-10, (f, err.max())


def test_star_steps_vs_oracle():
    from paper_2303_08058_b200.star import RotatingStarStep
    U, _ = so.initial_state(1)
    st = RotatingStarStep(1, device=torch.device("cuda", 0), state=torch.from_numpy(U))
    for k in range(3):
        U, dt = so.step(U, 1)
        st.step()
        assert abs(st.dt.item() - dt) <= 1e-12 * dt
        close(st.U.cpu().numpy(), U)


def test_star_graph_replay_equals_eager():
    from paper_2303_08058_b200.star import RotatingStarStep
    a = RotatingStarStep(2, device=torch.device("cuda", 0))
    b = RotatingStarStep(2, device=torch.device("cuda", 0))
    for _ in range(2):
        a.step()
        b.step(graph=True)
    torch.cuda.synchronize()
    assert torch.equal(a.U, b.U) and torch.equal(a.time, b.time)


def test_star_full_lattice_max_level_2():
    # every cell after 3 steps at max_level 2 (32^3 cells, 64 sub-grids)
    from paper_2303_08058_b200.star import RotatingStarStep
    U, _ = so.initial_state(2)
    st = RotatingStarStep(2, device=torch.device("cuda", 0), state=torch.from_numpy(U))
    for _ in range(3):
        U, dt = so.step(U, 2)
        st.step()
        assert abs(st.dt.item() - dt) <= 1e-12 * dt
        close(st.U.cpu().numpy(), U)


def sampled_subs(L, k=4, seed=0):
    n = 1 << L
    rng = np.random.default_rng(seed + L)
    centre = ((n // 2) * n + n // 2) * n + n // 2        # inside the star
    return np.unique(np.concatenate([[0, centre, n ** 3 - 1], rng.integers(0, n ** 3, k)]))


@pytest.mark.parametrize("L", [3, 4, 5])
def test_star_every_stage_sampled(L):
    """max_level 3-5 (the north_star's size): 3 steps; at each step both RK
    stages are checked on sampled sub-grids against the oracle fed the GPU's
    own state before that stage (hydro of the samples' ghosted blocks; FMM
    gravity at their cells, the oracle expanding only their ancestors);
    the stage-1 per-sub-grid amax on the samples, and dt exactly from the
    GPU's full amax."""
    from paper_2303_08058_b200.star import RotatingStarStep
    st = RotatingStarStep(L, device=torch.device("cuda", 0), record_stages=True)
    subs = sampled_subs(L)
    for _ in range(3):
        U0 = st.U.cpu().numpy()
        st.step()
        torch.cuda.synchronize()
        dt = st.dt.item()
        amax1 = st.amax1.cpu().numpy()
        U1, Un = st.U1.cpu().numpy(), st.U.cpu().numpy()
        assert dt == (st.cfl * st.dx) / amax1.max()
        L1, am, _ = so.sampled_rhs(U0, L, subs)
        assert np.all(np.abs(amax1[subs] - am) <= 1e-12 * am)
        u0 = so.blocks(U0, subs)
        close(np.moveaxis(so.blocks(U1, subs), 1, 0), np.moveaxis(u0 + dt * L1, 1, 0))
        L2, _, _ = so.sampled_rhs(U1, L, subs)
        want = 0.5 * (u0 + (so.blocks(U1, subs) + dt * L2))
        close(np.moveaxis(so.blocks(Un, subs), 1, 0), np.moveaxis(want, 1, 0))
        del U0, U1, Un


@pytest.mark.parametrize("L", [4, 5])
def test_star_conservation_budgets(L):
    """Whole-lattice identities of the spec at max_level 4-5: the hydro part
    conserves every field (periodic flux differences telescope), so per step
    mass is conserved, momentum changes by exactly the gravity impulse
    dt/2 (sum rho g at both stages) and energy by the gravity work
    dt/2 (sum s.g at both stages) — with the GPU's own stage states and g,
    to round-off of the lattice sums."""
    from paper_2303_08058_b200.star import RotatingStarStep
    st = RotatingStarStep(L, device=torch.device("cuda", 0), record_stages=True)

    def tot(x):
        return x.sum(dim=(-3, -2, -1))

    for _ in range(3):
        U0 = st.U.clone()
        st.step()
        torch.cuda.synchronize()
        dt = st.dt.item()
        d = tot(st.U) - tot(U0)                          # [5]
        scale = tot(U0.abs())
        assert abs(d[0].item()) <= 1e-13 * scale[0].item()
        imp = 0.5 * dt * (tot(U0[0] * st.g1) + tot(st.U1[0] * st.g2))        # [3]
        work = 0.5 * dt * (tot(U0[1:4] * st.g1).sum() + tot(st.U1[1:4] * st.g2).sum())
        gscale = 0.5 * dt * (tot((U0[0] * st.g1).abs()) + tot((st.U1[0] * st.g2).abs()))
        for c in range(3):
            assert abs(d[1 + c].item() - imp[c].item()) <= 1e-9 * gscale[c].item() + \
                1e-13 * scale[1 + c].item(), c
        assert abs(d[4].item() - work.item()) <= 1e-12 * scale[4].item()
    # the half-turn-symmetric star keeps (near) zero net momentum
    p = tot(st.U[1:4])
    assert (p.abs() <= 1e-10 * tot(st.U[1:4].abs())).all()


@pytest.mark.parametrize("n,nz,halo", [(8, 8, False), (16, 16, False), (24, 8, True),
                                       (16, 32, True), (40, 16, False)])
def test_pad_is_exact(n, nz, halo):
    """tb_star_pad_slab: x, y periodic, z from the neighbours' planes (or
    periodic without them) — an exact copy, checked against numpy."""
    from paper_2303_08058_b200 import _native as N
    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(n * 100 + nz)
    U = torch.rand((5, nz, n, n), dtype=torch.float64, generator=g)
    lo = torch.rand((5, 2, n, n), dtype=torch.float64, generator=g)
    hi = torch.rand((5, 2, n, n), dtype=torch.float64, generator=g)
    Up = torch.full((5, nz + 4, n + 4, n + 4), float("nan"), dtype=torch.float64, device=dev)
    Ud, lod, hid = U.to(dev), lo.to(dev), hi.to(dev)
    N.call("tb_star_pad_slab", 0, Ud.data_ptr(), n, nz, lod.data_ptr() if halo else None,
           hid.data_ptr() if halo else None, Up.data_ptr())
    torch.cuda.synchronize()
    u = U.numpy()
    if halo:
        u = np.concatenate([lo.numpy(), u, hi.numpy()], axis=1)
        want = np.pad(u, ((0, 0), (0, 0), (2, 2), (2, 2)), mode="wrap")
    else:
        want = np.pad(u, ((0, 0), (2, 2), (2, 2), (2, 2)), mode="wrap")
    np.testing.assert_array_equal(Up.cpu().numpy(), want)


def test_cfl_propagates_nan():
    # a sub-grid whose signal speed is NaN makes dt NaN (np.maximum / the
    # spec's amax.max()), instead of a finite dt from the others
    from paper_2303_08058_b200 import _native as N
    dev = torch.device("cuda", 0)
    amax = torch.linspace(0.5, 2.0, 3000, dtype=torch.float64, device=dev)
    dt = torch.zeros(1, dtype=torch.float64, device=dev)
    N.call("tb_star_cfl", 0, amax.data_ptr(), 3000, 0.01, 0.4, dt.data_ptr())
    torch.cuda.synchronize()
    assert dt.item() == (0.4 * 0.01) / 2.0
    amax[1234] = float("nan")
    N.call("tb_star_cfl", 0, amax.data_ptr(), 3000, 0.01, 0.4, dt.data_ptr())
    torch.cuda.synchronize()
    assert dt.isnan().item()
