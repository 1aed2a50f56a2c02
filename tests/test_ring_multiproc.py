"""Multi-rank host logic of the ring stepper on CPU (gloo, world_size 2 and 3):
partitioning, halo exchange ordering (incl. N=2 where both neighbours are
the same peer), exact accumulator all-reduce and min. The per-rank compute
is an oracle-backed CPU double of the five kernel primitives; the product
uses the same orchestration with libtb on NCCL."""

import math
import os
import socket
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import miniapp_oracle as mo
from paper_2303_08058_b200 import _native as N
from paper_2303_08058_b200.ring import RingStepper, ring_partition


def min_key(x: float) -> int:
    b = struct.unpack("<q", struct.pack("<d", x))[0]
    return b if b >= 0 else b ^ 0x7FFFFFFFFFFFFFFF


def key_to_double(k: int) -> float:
    b = k if k >= 0 else k ^ 0x7FFFFFFFFFFFFFFF
    return struct.unpack("<d", struct.pack("<q", b))[0]


class OracleRingOps:
    """CPU double of CudaRingOps (tests only): same data layout, same
    accumulator encoding (32-bit digits in int64 limbs + min key)."""

    def init_cells(self, cells, subgrids, lo):
        cells.copy_(torch.from_numpy(mo.initial_cells(subgrids, lo, lo + cells.shape[0])))

    def step(self, old, out, lf, rf, chains, kpc, acc, mins=None, sums=None):
        new, m, s = mo.step_cells(old.numpy(), lf.numpy().copy(), rf.numpy().copy(),
                                  chains, kpc)
        out.copy_(torch.from_numpy(new))
        limbs = acc[:N.TB_ACC_LIMBS].tolist()
        for v in s.tolist():
            mo.acc_add(limbs, v)
        acc[:N.TB_ACC_LIMBS] = torch.tensor(limbs, dtype=torch.int64)
        acc[N.TB_ACC_MIN_WORD] = min(int(acc[N.TB_ACC_MIN_WORD]), min_key(float(m.min())))
        if mins is not None:
            mins.copy_(torch.from_numpy(m))
            sums.copy_(torch.from_numpy(s))

    def acc_reset(self, acc):
        acc.zero_()
        acc[N.TB_ACC_MIN_WORD] = min_key(math.inf)

    def acc_finalize(self, acc, piece, dt, checksum):
        p = mo.acc_round([int(x) for x in acc[:N.TB_ACC_LIMBS].tolist()])
        piece[0] = p
        dt[0] = key_to_double(int(acc[N.TB_ACC_MIN_WORD]))
        checksum[0] = float(checksum[0]) + p
        self.acc_reset(acc)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, subgrids, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        st = RingStepper(subgrids, device=torch.device("cpu"), rank=rank, world=world,
                         max_steps=steps, ops=OracleRingOps())
        res = st.run(steps)
        q.put((rank, res.checksum, res.dts, st.lo, st.cells.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,subgrids,steps", [(2, 8, 2), (2, 3, 3), (3, 16, 3),
                                                  (3, 7, 2), (4, 4, 2), (4, 13, 2)])
def test_partitioned_ring_matches_single_device(world, subgrids, steps):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, subgrids, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cs, dts, cells = mo.run_reference_cells(subgrids, steps)
    for rank, got_cs, got_dts, lo, got_cells in outs:
        assert got_cs == cs and got_dts == dts
        np.testing.assert_array_equal(got_cells, cells[lo:lo + got_cells.shape[0]])


def test_single_rank_cpu_double_matches_golden(golden):
    st = RingStepper(4, device=torch.device("cpu"), max_steps=2, ops=OracleRingOps())
    res = st.run(2)
    lit = golden["reference_test_literals"]
    assert res.checksum == float.fromhex(lit["GOLDEN_4X2"])
    assert res.dts == [float.fromhex(h) for h in lit["GOLDEN_4X2_DTS"]]


def test_ring_partition_balanced_and_contiguous():
    for s in (2, 7, 8, 100, 32768 * 8 + 3):
        for w in (1, 2, 3, 8):
            if s < w:
                continue
            ranges = [ring_partition(s, w, r) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == s
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [h - l for l, h in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        ring_partition(1, 2, 0)


class _PeerStub:
    """The attributes RingStepper._map_peers reads, on CPU (tests only)."""

    def __init__(self, rank, world, fail):
        self.rank, self.world, self.group = rank, world, None
        self.device = torch.device("cpu")
        self.state = [torch.zeros(4, 512, dtype=torch.float64) for _ in range(2)]
        self.n = 4
        self.fail = fail

    def _export(self, t):
        if self.fail == ("export", self.rank):
            raise RuntimeError("export failed")
        return bytes(N.TB_IPC_HANDLE_BYTES), 0


def _map_worker(rank, world, port, fail, q):
    import paper_2303_08058_b200.ring as ring
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []

    def fake_call(name, *args):
        calls.append(name)
        if name == "tb_ipc_open_handle":
            if fail == ("open", rank):
                raise RuntimeError("open failed")
            args[1]._obj.value = 0x1000 * (len(calls) + 1)
        return 0

    ring.N.call = fake_call
    try:
        peers, err = RingStepper._map_peers(_PeerStub(rank, world, fail))
        q.put((rank, peers is not None, calls.count("tb_ipc_open_handle"),
               calls.count("tb_ipc_close")))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail", [None, ("export", 1), ("open", 1), ("open", 0)])
def test_peer_mapping_is_all_or_nothing(fail):
    """A rank whose IPC export or open fails must not leave the others on the
    peer-memory halo: every rank takes the same path (ring.py _map_peers)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_map_worker, args=(r, world, port, fail, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert {ok for _, ok, _, _ in outs} == {fail is None}
    for rank, ok, opens, closes in outs:
        # every successful open is closed again when any rank failed
        assert closes == (0 if ok else (opens if fail != ("open", rank) else opens - 1))
