"""Parity of the sm_100a kernels with the oracle (bit-exact), through the C ABI."""

import ctypes
import math

import numpy as np
import pytest

from conftest import fx
from oracle import miniapp_oracle as mo

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def N():
    from paper_2303_08058_b200 import _native
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    _native.init(0)
    return _native


def stream():
    return torch.cuda.current_stream().cuda_stream


def P(t):
    return t.data_ptr()


@pytest.mark.parametrize("kind", range(5))
@pytest.mark.parametrize("n", [1, 2, 3, 512, 4096 + 3, 1 << 20])
def test_transform_kinds_bit_exact(N, kind, n):
    rng = np.random.default_rng(kind * 1000 + n)
    host = rng.standard_normal(n + 1) * 10.0 ** rng.integers(-5, 5, n + 1)
    d = torch.from_numpy(host).cuda()
    view = d[1:]  # 8-byte aligned, not 16: exercises the unaligned head
    N.call("tb_transform", stream(), kind, P(view), n)
    want = host[1:].copy()
    mo.transform(want, kind)
    np.testing.assert_array_equal(view.cpu().numpy(), want)
    assert d[0].item() == host[0]      # untouched


def test_affine_and_noop(N):
    x = torch.arange(1000, dtype=torch.float64, device="cuda") * 0.37
    ref = x.cpu().numpy().copy()
    N.call("tb_launch", stream(), N.TB_OP_AFFINE, 0, 1.0, 1.0, P(x), 1000)
    np.testing.assert_array_equal(x.cpu().numpy(), ref + 1.0)
    N.call("tb_launch", stream(), N.TB_OP_NONE, 0, 1.0, 0.0, P(x), 1000)
    np.testing.assert_array_equal(x.cpu().numpy(), ref + 1.0)


def test_init_cells_matches_reference_init(N):
    for s, lo, n in [(4, 0, 4), (512, 0, 512), (4096, 1000, 77), (262144, 262000, 144)]:
        c = torch.empty((n, 512), dtype=torch.float64, device="cuda")
        N.call("tb_init_cells", stream(), P(c), s, lo, n)
        np.testing.assert_array_equal(c.cpu().numpy(), mo.initial_cells(s, lo, lo + n))


@pytest.mark.parametrize("s", [1, 2, 3, 8, 9, 64, 1000, 4096])
def test_fused_step_cells_mins_sums_bit_exact(N, s):
    old_h = mo.initial_cells(s)
    # perturb so faces differ from the closed form
    old_h = old_h + np.sin(np.arange(old_h.size)).reshape(old_h.shape) * 1e-3
    old = torch.from_numpy(old_h).cuda()
    out = torch.empty_like(old)
    mins = torch.empty(s, dtype=torch.float64, device="cuda")
    sums = torch.empty(s, dtype=torch.float64, device="cuda")
    acc = torch.zeros(N.TB_ACC_WORDS, dtype=torch.int64, device="cuda")
    N.call("tb_acc_reset", stream(), P(acc))
    N.call("tb_step", stream(), P(old), P(out), s, P(old[s - 1, 504:]), P(old[0, :8]),
           3, 5, P(mins), P(sums), P(acc))
    piece = torch.zeros(1, dtype=torch.float64, device="cuda")
    dt = torch.zeros(1, dtype=torch.float64, device="cuda")
    cs = torch.zeros(1, dtype=torch.float64, device="cuda")
    N.call("tb_acc_finalize", stream(), P(acc), P(piece), P(dt), P(cs), 1)
    want, wmin, wsum = mo.step_cells(old_h)
    np.testing.assert_array_equal(out.cpu().numpy(), want)
    np.testing.assert_array_equal(mins.cpu().numpy(), wmin)
    np.testing.assert_array_equal(sums.cpu().numpy(), wsum)
    assert piece.item() == math.fsum(wsum.tolist())
    assert dt.item() == float(wmin.min())
    assert cs.item() == piece.item()
    # reset re-armed the accumulator
    assert acc[:N.TB_ACC_LIMBS].abs().sum().item() == 0


def test_fused_step_explicit_halo_and_generic_chain(N):
    s = 33
    old_h = mo.initial_cells(100, 40, 40 + s)
    left = mo.initial_cells(100, 39, 40)[0, -8:].copy()
    right = mo.initial_cells(100, 73, 74)[0, :8].copy()
    old = torch.from_numpy(old_h).cuda()
    out = torch.empty_like(old)
    lt, rt = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
    for chains, kpc in [(3, 5), (2, 4), (1, 1), (0, 5)]:
        N.call("tb_step", stream(), P(old), P(out), s, P(lt), P(rt), chains, kpc,
               None, None, None)
        want, _, _ = mo.step_cells(old_h, left, right, chains, kpc)
        np.testing.assert_array_equal(out.cpu().numpy(), want)


def test_exact_accumulator_equals_fsum(N):
    rng = np.random.default_rng(3)
    acc = torch.zeros(N.TB_ACC_WORDS, dtype=torch.int64, device="cuda")
    out = torch.zeros(3, dtype=torch.float64, device="cuda")
    for trial in range(40):
        n = int(rng.integers(1, 200_000))
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
        if trial % 5 == 0:
            x = np.concatenate([x, -x[: n // 2]])     # heavy cancellation
        xt = torch.from_numpy(x).cuda()
        N.call("tb_acc_reset", stream(), P(acc))
        N.call("tb_acc_add", stream(), P(xt), x.size, P(acc))
        out.zero_()
        N.call("tb_acc_finalize", stream(), P(acc), P(out[0:1]), P(out[1:2]), None, 1)
        assert out[0].item() == math.fsum(x.tolist()), trial
        assert out[1].item() == x.min()
    for case in ([1.0, 2.0 ** -53], [1.0, 2.0 ** -53, 2.0 ** -106], [1e308, -1e308, 1.0],
                 [5e-324, 5e-324, -1e-323], [2.0 ** -1074] * 7, [-1.5, 2.0 ** -54],
                 [1.7976931348623157e308, -1.0]):
        xt = torch.tensor(case, dtype=torch.float64, device="cuda")
        N.call("tb_acc_reset", stream(), P(acc))
        N.call("tb_acc_add", stream(), P(xt), len(case), P(acc))
        N.call("tb_acc_finalize", stream(), P(acc), P(out[0:1]), None, None, 1)
        assert out[0].item() == math.fsum(case), case


@pytest.mark.parametrize("key", ["1x2", "3x3", "4x2", "8x2", "64x3", "512x1", "512x15",
                                 "4096x1", "32768x1", "262144x1"])
def test_ring_stepper_reproduces_reference_runs(N, golden, key):
    from paper_2303_08058_b200.ring import run_reference_gpu
    g = golden["run_reference"][key]
    cs, dts = run_reference_gpu(g["subgrids"], g["steps"])
    assert cs.hex() == g["checksum"]
    assert [d.hex() for d in dts] == g["dts"]


def test_ring_stepper_reference_literals(N, golden):
    from paper_2303_08058_b200.ring import RingStepper, run_reference_gpu
    lit = golden["reference_test_literals"]
    cs, dts = run_reference_gpu(4, 2)
    assert cs == fx(lit["GOLDEN_4X2"]) and dts == [fx(h) for h in lit["GOLDEN_4X2_DTS"]]
    assert run_reference_gpu(512, 15)[0] == fx(lit["GOLDEN_DEFAULTS"])
    st = RingStepper(16)
    st.run(3)
    cells = np.load(__import__("conftest").TESTS + "/golden/cells.npz")["cells_16x3"]
    np.testing.assert_array_equal(st.cells.cpu().numpy(), cells)


def test_ring_stepper_long_run_matches_c_oracle(N):
    from oracle import c_oracle
    from paper_2303_08058_b200.ring import run_reference_gpu
    cs, dts = run_reference_gpu(3000, 40)
    ccs, cdts = c_oracle.run_reference(3000, 40)
    assert cs == ccs and dts == cdts


@pytest.mark.parametrize("impl", ["reg", "bulk", "regpf", "lean", "pair", "bulk1"])
@pytest.mark.parametrize("s", [1, 5, 64, 3000])
def test_step_impls_and_fused_finalize(N, impl, s):
    code = {"reg": N.TB_STEP_REG, "bulk": N.TB_STEP_BULK, "regpf": N.TB_STEP_REGPF,
            "lean": N.TB_STEP_LEAN, "pair": N.TB_STEP_PAIR, "bulk1": N.TB_STEP_BULK1}[impl]
    N.call("tb_set_option", N.TB_OPT_STEP_IMPL, code)
    try:
        old_h = mo.initial_cells(s) + 1e-4 * np.cos(np.arange(s * 512)).reshape(s, 512)
        old = torch.from_numpy(old_h).cuda()
        out = torch.empty_like(old)
        acc = torch.zeros(N.TB_ACC_WORDS, dtype=torch.int64, device="cuda")
        res = torch.zeros(3, dtype=torch.float64, device="cuda")
        N.call("tb_acc_reset", stream(), P(acc))
        want, wmin, wsum = mo.step_cells(old_h)
        for rep in range(3):      # the ticket counter must re-arm every step
            res[2] = 0.0
            N.call("tb_step_final", stream(), P(old), P(out), s, P(old[s - 1, 504:]),
                   P(old[0, :8]), 3, 5, None, None, P(acc), P(res[0:1]), P(res[1:2]),
                   P(res[2:3]))
            np.testing.assert_array_equal(out.cpu().numpy(), want)
            assert res[0].item() == math.fsum(wsum.tolist())
            assert res[1].item() == float(wmin.min())
            assert res[2].item() == res[0].item()
        # generic chain through the same impl
        N.call("tb_step", stream(), P(old), P(out), s, P(old[s - 1, 504:]), P(old[0, :8]),
               2, 3, None, None, None)
        np.testing.assert_array_equal(out.cpu().numpy(), mo.step_cells(old_h, None, None,
                                                                       2, 3)[0])
    finally:
        N.call("tb_set_option", N.TB_OPT_STEP_IMPL, N.TB_STEP_AUTO)


@pytest.mark.parametrize("s,chunks", [(1, 4), (7, 3), (64, 16), (1000, 7), (4096, 16)])
def test_step_host_pipeline_matches_oracle(N, s, chunks):
    from paper_2303_08058_b200.ring import RingStepper
    st = RingStepper(s, max_steps=4)
    cells = torch.from_numpy(mo.initial_cells(s)).pin_memory()
    stats = torch.zeros(2, dtype=torch.float64).pin_memory()
    cs, dts, want = mo.run_reference_cells(s, 3)
    pieces = []
    for _ in range(3):
        st.step_host(cells, cells, stats, chunks=chunks, join=False)
        st.join_host()
        torch.cuda.synchronize()
        pieces.append(stats[0].item())
        assert stats[1].item() == dts[len(pieces) - 1]
    np.testing.assert_array_equal(cells.numpy(), want)
    assert st.result().checksum == cs


@pytest.mark.parametrize("spw", [1, 2, 5])
def test_step_grid_granularity(N, spw):
    N.call("tb_set_option", N.TB_OPT_STEP_SPW, spw)
    try:
        from paper_2303_08058_b200.ring import run_reference_gpu
        cs, dts = run_reference_gpu(4097, 2)
        ccs, cdts = mo.run_reference(4097, 2)
        assert cs == ccs and dts == cdts
    finally:
        N.call("tb_set_option", N.TB_OPT_STEP_SPW, 0)


def test_step_host_chained_unjoined_and_mixed_with_resident(N):
    from paper_2303_08058_b200.ring import RingStepper
    s = 777
    st = RingStepper(s, max_steps=16)
    cells = torch.from_numpy(mo.initial_cells(s)).pin_memory()
    stats = torch.zeros(2, dtype=torch.float64).pin_memory()
    for _ in range(4):                      # chained, never joined in between
        st.step_host(cells, cells, stats, chunks=5, join=False)
    st.join_host()
    torch.cuda.synchronize()
    cs, dts, want = mo.run_reference_cells(s, 4)
    np.testing.assert_array_equal(cells.numpy(), want)
    # host step without download, then resident steps continue from device state
    st.step_host(cells, None, stats, chunks=3)
    st.step()
    torch.cuda.synchronize()
    cs6, dts6, want6 = mo.run_reference_cells(s, 6)
    np.testing.assert_array_equal(st.cells.cpu().numpy(), want6)
    assert st.result().checksum == cs6 and st.result().dts == dts6


@pytest.mark.parametrize("world,subgrids", [(2, 64), (3, 100), (4, 4), (2, 3), (8, 1000)])
def test_partitioned_step_on_gpu_matches_single_device(N, world, subgrids):
    """The N>1 device path (interior K2 while the halo is in flight, then the
    two boundary sub-grids; limbs summed and min keys min-reduced across
    ranks) run for all ranks inside one process on one GPU, with the NCCL
    exchange and all-reduce replaced by in-process copies."""
    from paper_2303_08058_b200.ring import CELLS, FACE, RingStepper
    ranks = [RingStepper(subgrids, rank=r, world=world, max_steps=4) for r in range(world)]
    for st in ranks:
        st._exchange_start = lambda *a, **k: []      # halo filled below

    for _ in range(3):
        olds = [st.state[st.cur] for st in ranks]
        for r, st in enumerate(ranks):
            left, right = ranks[(r - 1) % world], ranks[(r + 1) % world]
            st.halo[0].copy_(olds[(r - 1) % world][left.n - 1, CELLS - FACE:])
            st.halo[1].copy_(olds[(r + 1) % world][0, :FACE])
        for st in ranks:
            st._step_partitioned(st.state[st.cur], st.state[1 - st.cur], None)
        limbs = sum(st.acc[:N.TB_ACC_LIMBS] for st in ranks)
        mkey = torch.stack([st.acc[N.TB_ACC_MIN_WORD] for st in ranks]).min()
        for st in ranks:
            st.acc[:N.TB_ACC_LIMBS].copy_(limbs)
            st.acc[N.TB_ACC_MIN_WORD] = mkey
            k = st.steps_done
            st.ops.acc_finalize(st.acc, st.pieces[k:k + 1], st.dts[k:k + 1], st.checksum)
            st.cur = 1 - st.cur
            st.steps_done += 1
    cs, dts, cells = mo.run_reference_cells(subgrids, 3)
    for st in ranks:
        res = st.result()
        assert res.checksum == cs and res.dts == dts
        np.testing.assert_array_equal(st.cells.cpu().numpy(), cells[st.lo:st.hi])


def test_step_host_inplace_chain_faces_from_device(N):
    from paper_2303_08058_b200.ring import RingStepper
    for s, chunks in [(1, 1), (2, 2), (500, 7)]:
        st = RingStepper(s, max_steps=8)
        cells = torch.from_numpy(mo.initial_cells(s)).pin_memory()
        stats = torch.zeros(2, dtype=torch.float64).pin_memory()
        for _ in range(5):
            st.step_host(cells, cells, stats, chunks=chunks, join=False)
        st.join_host()
        torch.cuda.synchronize()
        cs, dts, want = mo.run_reference_cells(s, 5)
        np.testing.assert_array_equal(cells.numpy(), want)
        assert st.result().checksum == cs and st.result().dts == dts
