"""Self-authored hydro oracle (PARITY UNPINNED — no hydro in the reference):
the physics properties any correct finite-volume flux kernel must have."""

import numpy as np
import pytest

from oracle import hydro_oracle as h


def test_uniform_state_has_zero_update():
    U = np.empty((3, 5, 12, 12, 12))
    U[:, 0], U[:, 1], U[:, 2], U[:, 3], U[:, 4] = 1.3, 0.2, -0.1, 0.05, 4.0
    du, amax = h.hydro_flux(U, 0.01, 5 / 3)
    assert np.all(du == 0.0)
    rho, v = 1.3, np.array([0.2, -0.1, 0.05]) / 1.3
    p = (5 / 3 - 1) * (4.0 - 0.5 * 1.3 * (v @ v))
    assert np.allclose(amax, np.abs(v).max() + np.sqrt(5 / 3 * p / rho), rtol=1e-12)


@pytest.mark.parametrize("s", [8, 27])
def test_conservation_on_periodic_lattice(s):
    I, dx = h.rotating_star(s)
    du, _ = h.hydro_flux(h.with_ghosts(I), dx, 5 / 3)
    tot = du.sum(axis=(0, 2, 3, 4))
    mag = np.abs(du).sum(axis=(0, 2, 3, 4))
    assert np.all(np.abs(tot) <= 1e-13 * mag + 1e-300)


def test_ghosts_match_neighbours():
    I, _ = h.rotating_star(8)
    U = h.with_ghosts(I)
    # interior of the ghosted block is the sub-grid itself
    np.testing.assert_array_equal(U[:, :, 2:10, 2:10, 2:10], I)
    # sub-grid 0's +x ghosts are sub-grid 1's first cells (x fastest)
    np.testing.assert_array_equal(U[0, :, 2:10, 2:10, 10:12], I[1, :, :, :, 0:2])


def test_mirror_symmetry():
    rng = np.random.default_rng(2)
    I, dx = h.rotating_star(8)
    I = I * (1 + 0.01 * rng.standard_normal(I.shape))
    U = h.with_ghosts(I)
    du, a = h.hydro_flux(U, dx, 5 / 3)
    Um = U[..., ::-1].copy()                 # mirror x within each sub-grid
    Um[:, 1] *= -1
    dum, am = h.hydro_flux(Um, dx, 5 / 3)
    want = du[..., ::-1].copy()
    want[:, 1] *= -1
    np.testing.assert_allclose(dum, want, rtol=1e-12, atol=1e-12 * np.abs(du).max())
    np.testing.assert_allclose(am, a, rtol=1e-14)


def test_positive_pressure_and_signal_speed():
    I, dx = h.rotating_star(27)
    rho, vx, vy, vz, p = h.primitives(h.with_ghosts(I), 5 / 3)
    assert (p > 0).all() and (rho > 0).all()
    _, a = h.hydro_flux(h.with_ghosts(I), dx, 5 / 3)
    assert (a > 0).all()


def test_product_synthetic_inputs_match_the_oracle_generator():
    torch = pytest.importorskip("torch")
    from paper_2303_08058_b200 import hydro
    for s in (1, 8, 27):
        I, dx = h.rotating_star(s)
        It, dxt = hydro.rotating_star(s)
        assert dx == dxt
        np.testing.assert_allclose(It.numpy(), I, rtol=1e-15, atol=1e-15)
        np.testing.assert_array_equal(hydro.with_ghosts(torch.from_numpy(I)).numpy(),
                                      h.with_ghosts(I))
