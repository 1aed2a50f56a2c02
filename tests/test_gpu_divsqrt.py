"""The branch-free FP64 division / square-root fast paths that K6 uses
(tb_internal.h div_rn_fast / sqrt_rn_fast, the IEEE intrinsic where they
flag) equal IEEE round-to-nearest division and square root bit for bit —
checked against numpy (the hydro oracle's arithmetic) over random bit
patterns of every class and over the magnitudes the hydro states take."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _run(a, b):
    from paper_2303_08058_b200 import _native as N
    N.init(0)
    da = torch.from_numpy(a).cuda()
    db = torch.from_numpy(b).cuda()
    q = torch.empty_like(da)
    r = torch.empty_like(da)
    slow = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert N.call("tb_divsqrt_fast", st, da.data_ptr(), db.data_ptr(), len(a), q.data_ptr(),
                  r.data_ptr(), slow.data_ptr()) == 0
    torch.cuda.synchronize()
    return q.cpu().numpy(), r.cpu().numpy(), int(slow.item())


def _same(x, y):
    return (x.view(np.int64) == y.view(np.int64)) | (np.isnan(x) & np.isnan(y))


def test_fast_paths_equal_ieee_on_random_bit_patterns():
    rng = np.random.default_rng(7)
    n = 1 << 22
    a = rng.integers(0, 2 ** 63, n, dtype=np.int64).view(np.float64).copy()
    b = rng.integers(0, 2 ** 63, n, dtype=np.int64).view(np.float64).copy()
    a[: n // 2] = np.abs(a[: n // 2])
    b[::3] = -b[::3]
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 2.2250738585072014e-308,
                        1.7976931348623157e308, 1.0, -1.0])
    a[: special.size ** 2] = np.repeat(special, special.size)
    b[: special.size ** 2] = np.tile(special, special.size)
    q, r, slow = _run(a, b)
    with np.errstate(all="ignore"):
        assert _same(q, a / b).all()
        assert _same(r, np.sqrt(a)).all()
    assert slow > 0          # the flagged domain is exercised too


def test_fast_paths_equal_ieee_on_hydro_magnitudes():
    rng = np.random.default_rng(8)
    n = 1 << 23
    a = 10.0 ** rng.uniform(-12, 12, n)
    b = 10.0 ** rng.uniform(-12, 12, n)
    q, r, slow = _run(a, b)
    assert (q.view(np.int64) == (a / b).view(np.int64)).all()
    assert (r.view(np.int64) == np.sqrt(a).view(np.int64)).all()
    assert slow == 0         # physical ranges never leave the fast path
