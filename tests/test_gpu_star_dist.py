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


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, L, steps, q):
    import os

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2303_08058_b200.star import RotatingStarStep
        from paper_2303_08058_b200.star_dist import DistDriver, StarSlab, split_state
        U = RotatingStarStep(L, device=torch.device("cuda", 0)).U
        slab = StarSlab(L, world, rank, split_state(U, world)[rank])
        drv = DistDriver(slab)
        for _ in range(steps):
            drv.step()
        torch.cuda.synchronize()
        # numpy travels by value (a shared torch tensor's file descriptor dies
        # with this process if it exits before the parent has read it)
        q.put((rank, slab.U.cpu().numpy(), slab.time.item()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,L", [(2, 2), (4, 3)])
def test_dist_driver_processes_equal_single_device(world, L):
    """torch.distributed orchestration (gloo + host staging, processes
    sharing one GPU): the gathered slabs equal the single-device step."""
    import torch.multiprocessing as mp

    from paper_2303_08058_b200.star import RotatingStarStep
    steps = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        outs = sorted([q.get(timeout=240) for _ in range(world)], key=lambda o: o[0])
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    ref = RotatingStarStep(L, device=torch.device("cuda", 0))
    for _ in range(steps):
        ref.step()
    got = torch.cat([torch.from_numpy(o[1]) for o in outs], dim=1)
    assert torch.equal(got, ref.U.cpu())
    assert all(o[2] == ref.time.item() for o in outs)
