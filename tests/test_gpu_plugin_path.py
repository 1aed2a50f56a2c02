"""The reference-facing call path (build_scenario + Runtime + CudaDevice +
Integration + ExecutorPool + AggregationExecutor + run_scenario, as
src/cli.py:199-232 wires it) delegated to libtb's native machine: goldens in
every completion mode, the reference's unfused counts, the aggregation
executors' counters, BASELINE config 4, and the configurations that must stay
on the Python machine."""

import numpy as np
import pytest

from conftest import fx

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")

from paper_2303_08058_b200 import (AggregationExecutor, BufferPool, CudaDevice,  # noqa: E402
                                   ExecutorPool, Integration, IntegrationMode, Runtime,
                                   ScenarioConfig, build_scenario, kernel_transform,
                                   run_scenario)

MODES = list(IntegrationMode)


class Rig:
    def __init__(self, workers=4, executors=2, max_agg=8, mode=IntegrationMode.POLLING, **dev):
        self.runtime = Runtime(workers)
        self.device = CudaDevice(0, **dev)
        integ = Integration(self.runtime, self.device, mode)
        pool = ExecutorPool(integ, executors)
        buffers = BufferPool(self.device)
        self.aggs = [AggregationExecutor(ex, max_agg, buffers) for ex in pool.executors]
        for a in self.aggs:
            for k in range(5):
                a.register_kind(k, kernel_transform(k))

    def run(self, subgrids, steps, by_grid=None, **kw):
        sc = build_scenario(ScenarioConfig(subgrids=subgrids, steps=steps))
        if by_grid is None:
            by_grid = [self.aggs[g % len(self.aggs)] for g in range(subgrids)]
        return sc, run_scenario(sc, self.runtime, self.device, self.aggs, by_grid, **kw)

    def close(self):
        self.runtime.shutdown()
        self.device.destroy()


@pytest.fixture
def rig():
    made = []

    def make(**kw):
        r = Rig(**kw)
        made.append(r)
        return r

    yield make
    for r in made:
        r.close()


@pytest.mark.parametrize("copies", ["staged", "gather", "resident", "direct"])
@pytest.mark.parametrize("mode", MODES)
def test_delegated_goldens_every_mode(rig, golden, mode, copies):
    lit = golden["reference_test_literals"]
    r = rig(workers=2, executors=2, max_agg=8, mode=mode)
    sc, res = r.run(4, 2, batch_copies=copies)
    assert res.engine == "native" and res.batch_copies == copies and sc.pinned
    assert res.checksum == fx(lit["GOLDEN_4X2"])
    assert res.dts == [fx(h) for h in lit["GOLDEN_4X2_DTS"]]
    r2 = rig(workers=4, executors=3, max_agg=4, mode=mode)
    sc, res = r2.run(16, 3, batch_copies=copies)
    assert res.engine == "native"
    assert res.checksum.hex() == golden["machine"]["16x3"]["checksum"]
    cells = np.load(__import__("conftest").TESTS + "/golden/cells.npz")["cells_16x3"]
    np.testing.assert_array_equal(sc.cells(), cells)


@pytest.mark.parametrize("mode", [IntegrationMode.POLLING, IntegrationMode.FENCE])
def test_delegated_completion_words(rig, golden, mode):
    r = rig(workers=4, executors=3, max_agg=4, mode=mode)
    sc, res = r.run(16, 3, batch_copies="direct", completion="words")
    assert res.engine == "native" and res.batch_copies == "direct"
    assert res.checksum.hex() == golden["machine"]["16x3"]["checksum"]
    cells = np.load(__import__("conftest").TESTS + "/golden/cells.npz")["cells_16x3"]
    np.testing.assert_array_equal(sc.cells(), cells)
    with pytest.raises(ValueError):     # staged batches end in a copy, not a kernel
        r.run(16, 1, batch_copies="staged", completion="words")


def test_fused_engine_goldens(rig, golden):
    """engine='fused': one K2 launch of all sub-grids per step through
    run_scenario — the reference's literals, cells and C4."""
    lit = golden["reference_test_literals"]
    r = rig(workers=2, executors=2, max_agg=8)
    for _ in range(2):           # the second call reuses the cached stepper
        sc, res = r.run(4, 2, engine="fused")
        assert res.engine == "fused"
        assert res.checksum == fx(lit["GOLDEN_4X2"])
        assert res.dts == [fx(h) for h in lit["GOLDEN_4X2_DTS"]]
    r2 = rig(workers=4, executors=3, max_agg=4)
    sc, res = r2.run(16, 3, engine="fused")
    assert res.checksum.hex() == golden["machine"]["16x3"]["checksum"]
    cells = np.load(__import__("conftest").TESTS + "/golden/cells.npz")["cells_16x3"]
    np.testing.assert_array_equal(sc.cells(), cells)
    r3 = rig(workers=4, executors=8, max_agg=64)
    _, res = r3.run(32768, 1, engine="fused")
    g = golden["run_reference"]["32768x1"]
    assert res.checksum.hex() == g["checksum"] and [d.hex() for d in res.dts] == g["dts"]
    assert res.per_step[0].launches == 1
    from paper_2303_08058_b200.miniapp import release_fused
    release_fused()


def test_delegated_unfused_counts_and_agg_counters(rig, golden):
    # pkg/tests/test_miniapp.py:65-75 on the delegated path
    r = rig(executors=1, max_agg=1)
    _, res = r.run(8, 2)
    assert res.engine == "native"
    for m in res.per_step:
        assert m.launches == 8 * 15 and m.transfers == 8 * 30
        assert sum(m.batch_sizes) == 120 and len(m.batch_sizes) == 120
        assert m.reasons_full == 120 and m.reasons_idle == 0 and m.event_waits == 0
    a = r.aggs[0]
    assert a.launches == 240 and sum(a.batch_sizes) == 240 and a.reasons["full"] == 240
    assert res.checksum == fx(golden["reference_test_literals"]["GOLDEN_8X2"])


def test_delegated_criterion1_and_fused_batches(rig, golden):
    r = rig(workers=8, executors=32, max_agg=1)
    _, res = r.run(512, 1)
    want = golden["machine_counts_512x1_m1"]
    assert res.per_step[0].launches == want["kernels"] == 7680
    assert res.per_step[0].transfers == want["transfers"] == 15360
    assert res.checksum.hex() == want["checksum"]
    r2 = rig(executors=1, max_agg=4)
    _, res = r2.run(8, 2)
    assert sum(sz for m in res.per_step for sz in m.batch_sizes) == 8 * 15 * 2
    assert max(sz for m in res.per_step for sz in m.batch_sizes) <= 4


def test_python_machine_when_not_delegable(rig, golden):
    lit = golden["reference_test_literals"]
    # a non-round-robin sub-grid -> executor map
    r = rig(executors=2)
    _, res = r.run(4, 2, by_grid=[r.aggs[0], r.aggs[0], r.aggs[1], r.aggs[1]])
    assert res.engine == "python" and res.checksum == fx(lit["GOLDEN_4X2"])
    with pytest.raises(ValueError):
        r.run(4, 2, by_grid=[r.aggs[0]] * 4, engine="native")
    # a lazy-submit device (the Python machine's flush hook)
    r2 = rig(lazy_submit=True)
    _, res = r2.run(4, 2)
    assert res.engine == "python" and res.checksum == fx(lit["GOLDEN_4X2"])
    # forced
    r3 = rig()
    _, res = r3.run(4, 2, engine="python")
    assert res.engine == "python" and res.checksum == fx(lit["GOLDEN_4X2"])


@pytest.mark.parametrize("mode", MODES)
def test_delegated_c4_golden(rig, golden, mode):
    g = golden["run_reference"]["32768x1"]
    r = rig(workers=16, executors=8, max_agg=256, mode=mode)
    _, res = r.run(32768, 1, batch_copies="gather")
    assert res.engine == "native"
    assert res.checksum.hex() == g["checksum"]
    assert [d.hex() for d in res.dts] == g["dts"]
