"""The multi-GPU peer-memory halo (CUDA IPC mapped neighbour state, ghost
faces read inside K2) exercised with 2 and 3 processes sharing one GPU: the
IPC mapping, pointer arithmetic into the neighbour's generation and the
all-reduce ordering argument are the same as across NVLink."""

import os
import socket

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, subgrids, steps, q, halo="p2p"):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2303_08058_b200.ring import RingStepper
        st = RingStepper(subgrids, device=torch.device("cuda", 0), rank=rank, world=world,
                         max_steps=steps, halo=halo)
        mode = st.halo_mode
        res = st.run(steps)
        cells = st.cells.cpu().numpy()
        dist.barrier()
        st.close()
        q.put((rank, mode, res.checksum, res.dts, st.lo, cells))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("halo", ["p2p", "nccl"])
@pytest.mark.parametrize("world,subgrids,steps", [(2, 64, 3), (3, 1000, 2), (2, 3, 2)])
def test_p2p_halo_ring_matches_reference(world, subgrids, steps, halo):
    """halo="nccl" here runs the message-passing path's orchestration on
    device buffers (gloo stages the faces through the host: several ranks
    cannot share one GPU under NCCL)."""
    import numpy as np
    import torch.multiprocessing as mp

    from oracle import miniapp_oracle as mo
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, subgrids, steps, q, halo))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        outs = [q.get(timeout=120) for _ in range(world)]
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    cs, dts, cells = mo.run_reference_cells(subgrids, steps)
    for rank, mode, got_cs, got_dts, lo, got in outs:
        assert mode == halo
        assert got_cs == cs and got_dts == dts
        np.testing.assert_array_equal(got, cells[lo:lo + got.shape[0]])
