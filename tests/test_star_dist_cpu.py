"""Exchange semantics of the slab-decomposed star step, on CPU: the
in-process VirtualCluster servicing and the torch.distributed DistDriver
(gloo, world 2 and 3) deliver the same halo planes, gathered slices and
minimum for fake slabs (no kernels involved)."""

import os
import socket

import pytest

torch = pytest.importorskip("torch")


def _reqs(R, kind, periodic=True):
    out = []
    for r in range(R):
        if kind == "halo":
            lo = torch.full((2, 3), 10.0 * r + 1)          # my lowest planes
            hi = torch.full((2, 3), 10.0 * r + 2)          # my highest planes
            out.append(("halo", lo, hi, torch.zeros(2, 3), torch.zeros(2, 3), periodic))
        elif kind == "allgather":
            full = torch.zeros(4 * R)
            full[4 * r:4 * r + 4] = r + 1.0
            out.append(("allgather", full, 4 * r, 4 * r + 4))
        else:
            out.append(("min", torch.tensor([5.0 - r])))
    return out


@pytest.mark.parametrize("R", [1, 2, 3])
@pytest.mark.parametrize("periodic", [True, False])
def test_virtual_halo_service(R, periodic):
    from paper_2303_08058_b200.star_dist import VirtualCluster
    vc = VirtualCluster.__new__(VirtualCluster)
    vc.ranks = R
    reqs = _reqs(R, "halo", periodic)
    vc._service(reqs)
    for r, (_, _, _, rlo, rhi, _) in enumerate(reqs):
        if periodic or r > 0:
            assert torch.all(rlo == 10.0 * ((r - 1) % R) + 2)     # neighbour below's top
        else:
            assert torch.all(rlo == 0)
        if periodic or r < R - 1:
            assert torch.all(rhi == 10.0 * ((r + 1) % R) + 1)     # neighbour above's bottom
        else:
            assert torch.all(rhi == 0)


def test_virtual_allgather_and_min():
    from paper_2303_08058_b200.star_dist import VirtualCluster
    vc = VirtualCluster.__new__(VirtualCluster)
    vc.ranks = 3
    reqs = _reqs(3, "allgather")
    vc._service(reqs)
    for q in reqs:
        assert torch.equal(q[1], torch.repeat_interleave(torch.tensor([1.0, 2.0, 3.0]), 4))
    reqs = _reqs(3, "min")
    vc._service(reqs)
    assert all(q[1].item() == 3.0 for q in reqs)


class _FakeSlab:
    def __init__(self, R, r):
        self.R, self.r = R, r


def test_virtual_wait_is_a_no_op():
    from paper_2303_08058_b200.star_dist import VirtualCluster
    vc = VirtualCluster.__new__(VirtualCluster)
    vc.ranks = 2
    vc._service([("wait", 0), ("wait", 0)])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2303_08058_b200.star_dist import DistDriver
        drv = DistDriver(_FakeSlab(world, rank))
        res = {}
        for periodic in (True, False):
            _, lo, hi, rlo, rhi, _ = _reqs(world, "halo", periodic)[rank]
            drv._halo(lo, hi, rlo, rhi, periodic)
            drv._wait(first_only=False)
            res[periodic] = (rlo.clone(), rhi.clone())
        _, full, a, b = _reqs(world, "allgather")[rank]
        drv._allgather(full, a, b)
        drv._wait(first_only=False)
        m = _reqs(world, "min")[rank][1]
        drv._min(m)
        # numpy payloads travel by value (a torch tensor would be shared through
        # a file descriptor that dies with this process if it exits first)
        q.put((rank, {k: (a.numpy(), b.numpy()) for k, (a, b) in res.items()},
               full.numpy().copy(), m.item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dist_driver_matches_virtual_cluster(world):
    import torch.multiprocessing as mp

    from paper_2303_08058_b200.star_dist import VirtualCluster
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        outs = sorted([q.get(timeout=120) for _ in range(world)], key=lambda o: o[0])
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    vc = VirtualCluster.__new__(VirtualCluster)
    vc.ranks = world
    for periodic in (True, False):
        want = _reqs(world, "halo", periodic)
        vc._service(want)
        for r in range(world):
            assert torch.equal(torch.from_numpy(outs[r][1][periodic][0]), want[r][3])
            assert torch.equal(torch.from_numpy(outs[r][1][periodic][1]), want[r][4])
    gathered = torch.repeat_interleave(torch.arange(1.0, world + 1), 4)
    assert all(torch.equal(torch.from_numpy(o[2]), gathered) for o in outs)
    assert all(o[3] == 5.0 - (world - 1) for o in outs)
