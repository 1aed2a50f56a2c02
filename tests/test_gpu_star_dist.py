"""The rotating-star step split into z-slabs (PARITY UNPINNED against the
reference, which has no physics): any number of ranks reproduces the
single-device step bit for bit, because the partitioned step is the same
arithmetic on the same operands (halo planes and gathered records carry the
exact neighbour values; the CFL dt is an exact min)."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("L,R", [(2, 1), (2, 2), (3, 2), (3, 4), (4, 8)])
def test_virtual_cluster_equals_single_device(L, R):
    from paper_2303_08058_b200.star import RotatingStarStep
    from paper_2303_08058_b200.star_dist import VirtualCluster
    dev = torch.device("cuda", 0)
    ref = RotatingStarStep(L, device=dev)
    vc = VirtualCluster(L, R, ref.U.clone())
    for _ in range(2):
        ref.step()
        vc.step()
    torch.cuda.synchronize()
    assert torch.equal(vc.state(), ref.U)
    assert all(torch.equal(s.time, ref.time) for s in vc.slabs)


def test_slab_rejects_bad_geometry():
    from paper_2303_08058_b200.star_dist import StarSlab
    U = torch.zeros((5, 8, 32, 32), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        StarSlab(2, 4, 0, U)          # 32 / 4 = 8 planes < one 16-plane leaf tile
