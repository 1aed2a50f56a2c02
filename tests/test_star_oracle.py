"""Self-authored coupled rotating-star step (PARITY UNPINNED — the reference
has no physics): properties of the spec, on CPU."""

import numpy as np
import pytest

from oracle import star_oracle as so


def test_layout_round_trip():
    U, _ = so.initial_state(1)
    assert np.array_equal(so.subgrids_to_lattice(so.lattice_to_subgrids(U)), U)


def test_step_conserves_mass_and_total_momentum():
    U, dx = so.initial_state(1)
    U2, dt = so.step(U, 1)
    assert dt > 0 and np.isfinite(U2).all()
    m0, m1 = U[0].sum(), U2[0].sum()
    assert abs(m1 - m0) <= 1e-14 * m0
    # the star is symmetric under a half turn about z: total momentum stays 0
    for a in (1, 2, 3):
        assert abs(U2[a].sum()) <= 1e-12 * np.abs(U2[a]).sum()
    assert not np.array_equal(U2, U)


def test_product_layout_helper_matches_the_oracle():
    torch = pytest.importorskip("torch")
    from paper_2303_08058_b200.star import subgrids_to_lattice
    from oracle import hydro_oracle as ho
    I, _ = ho.rotating_star(8)
    assert np.array_equal(subgrids_to_lattice(torch.from_numpy(I)).numpy(),
                          so.subgrids_to_lattice(I))


def test_sampled_rhs_equals_full_oracle():
    # the full-size GPU checks (tests/test_gpu_star.py) rest on this: L(U)
    # restricted to sampled sub-grids == the full oracle's rows, bit for bit
    import numpy as np
    from oracle import star_oracle as so
    for L, subs in ((1, [0, 3, 5, 7]), (2, [0, 9, 36, 63])):
        U, _ = so.initial_state(L)
        U = U * (1.0 + 1e-3 * np.sin(np.arange(U.size)).reshape(U.shape))
        full, am = so.rhs(U, L, 5 / 3)
        Ls, ams, _ = so.sampled_rhs(U, L, np.array(subs))
        assert np.array_equal(Ls, so.lattice_to_subgrids(full)[subs])
        assert np.array_equal(ams, am[subs])
