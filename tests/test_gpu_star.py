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


def test_star_conserves_mass_at_max_level_4():
    from paper_2303_08058_b200.star import RotatingStarStep
    st = RotatingStarStep(4, device=torch.device("cuda", 0))
    m0, p0, _ = st.totals()
    for _ in range(2):
        st.step()
    m1, p1, _ = st.totals()
    assert abs(m1 - m0) <= 1e-13 * m0
    assert torch.isfinite(st.U).all()
    assert st.dt.item() > 0


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
