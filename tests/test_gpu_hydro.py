"""K6 hydro reconstruct+flux on the GPU: bit-identical to the self-authored
oracle (PARITY UNPINNED against the reference, which has no hydro) and
conservative to round-off at the BASELINE config-2 size."""

import numpy as np
import pytest

from oracle import hydro_oracle as h

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("s,seed", [(1, 0), (8, 1), (27, 2), (64, 3)])
def test_hydro_flux_bit_exact_vs_oracle(s, seed):
    from paper_2303_08058_b200.hydro import hydro_flux
    rng = np.random.default_rng(seed)
    I, dx = h.rotating_star(s)
    I = I * (1 + 0.05 * rng.standard_normal(I.shape))
    I[:, 4] = np.abs(I[:, 4]) + 0.5          # keep the pressure positive
    I[:, 0] = np.abs(I[:, 0]) + 1e-3
    U = h.with_ghosts(I)
    want, wa = h.hydro_flux(U, dx, 5 / 3)
    got, ga = hydro_flux(torch.from_numpy(U).cuda(), dx, 5 / 3)
    np.testing.assert_array_equal(got.cpu().numpy(), want)
    np.testing.assert_array_equal(ga.cpu().numpy(), wa)


def test_hydro_flux_uniform_and_conservation_at_c2_size():
    from paper_2303_08058_b200.hydro import hydro_flux
    I, dx = h.rotating_star(4096)                 # 16^3 sub-grids = config 2 batch
    U = torch.from_numpy(h.with_ghosts(I)).cuda()
    du, a = hydro_flux(U, dx)
    du = du.cpu().numpy()
    tot = du.sum(axis=(0, 2, 3, 4))
    mag = np.abs(du).sum(axis=(0, 2, 3, 4))
    assert np.all(np.abs(tot) <= 1e-12 * mag)
    assert torch.isfinite(a).all() and (a > 0).all()
    Uu = torch.empty((5, 5, 12, 12, 12), dtype=torch.float64, device="cuda")
    for f, v in enumerate((1.0, 0.1, 0.2, 0.3, 5.0)):
        Uu[:, f] = v
    duu, _ = hydro_flux(Uu, 0.1)
    assert (duu == 0).all()
