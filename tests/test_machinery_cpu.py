"""Host logic of the reference-facing machine on CPU, with a test double of
the device (tests/fake_device.py): Integration modes, executors, aggregation
partitioning, the mini-app's goldens and counts (pkg/tests/test_miniapp.py,
test_executors.py, test_bridge.py, acceptance criteria 1, 2, 6, 7)."""

import random
import threading

import numpy as np
import pytest

from conftest import fx
from fake_device import FakeDevice
from oracle import miniapp_oracle as mo
from paper_2303_08058_b200 import (AggregationExecutor, BufferPool, DeviceGoneError,
                                   ExecutorPool, FutureStatus, Integration,
                                   IntegrationMode, KindError, OrderingError, PoolError,
                                   Runtime, ScenarioConfig, StateError, affine_kernel,
                                   build_scenario, kernel_transform, make_dummy,
                                   make_spin, run_scenario, when_all)
from paper_2303_08058_b200.miniapp import _min_tree
from paper_2303_08058_b200.runtime import make_promise

MODES = list(IntegrationMode)


class Stack:
    def __init__(self, workers=2, mode=IntegrationMode.POLLING, executors=1, max_agg=4,
                 inject_barriers=True, barrier_elision=False, op_delay=0.0):
        self.runtime = Runtime(workers, seed=7)
        self.device = FakeDevice(op_delay=op_delay, barrier_elision=barrier_elision)
        self.integration = Integration(self.runtime, self.device, mode)
        self.executors = ExecutorPool(self.integration, executors)
        self.buffers = BufferPool(self.device)
        self.aggs = [AggregationExecutor(ex, max_agg, self.buffers,
                                         inject_barriers=inject_barriers)
                     for ex in self.executors.executors]
        for a in self.aggs:
            for k in range(5):
                a.register_kind(k, kernel_transform(k))

    def close(self):
        self.runtime.shutdown()
        self.device.destroy()


@pytest.fixture
def stacks():
    made = []

    def make(**kw):
        s = Stack(**kw)
        made.append(s)
        return s

    yield make
    for s in made:
        s.close()


def run(stack, s, n):
    sc = build_scenario(ScenarioConfig(subgrids=s, steps=n))
    by_grid = [stack.aggs[i % len(stack.aggs)] for i in range(s)]
    return sc, run_scenario(sc, stack.runtime, stack.device, stack.aggs, by_grid)


@pytest.mark.parametrize("mode", MODES)
def test_goldens_every_mode(stacks, golden, mode):
    lit = golden["reference_test_literals"]
    s = stacks(workers=2, executors=2, max_agg=8, mode=mode)
    _, res = run(s, 4, 2)
    assert res.checksum == fx(lit["GOLDEN_4X2"])
    assert res.dts == [fx(h) for h in lit["GOLDEN_4X2_DTS"]]
    sc, res = run(stacks(workers=4, executors=3, max_agg=4, mode=mode), 16, 3)
    assert res.checksum.hex() == golden["machine"]["16x3"]["checksum"]
    cells = np.load(__import__("conftest").TESTS + "/golden/cells.npz")["cells_16x3"]
    np.testing.assert_array_equal(sc.cells(), cells)


def test_unfused_counts(stacks, golden):
    s = stacks(executors=1, max_agg=1)
    _, res = run(s, 8, 2)
    for m in res.per_step:
        assert m.launches == 120 and m.transfers == 240
        assert m.reasons_full == 120 and m.reasons_idle == 0 and m.event_waits == 0
    assert res.checksum == fx(golden["reference_test_literals"]["GOLDEN_8X2"])


def test_criterion2_matrix_subset(golden):
    want = fx(golden["reference_test_literals"]["GOLDEN_8X2"]).hex()
    seen = set()
    for mode in MODES:
        for e, m, w, elide in [(1, 1, 1, False), (8, 8, 4, True), (32, 32, 8, False),
                               (8, 1, 8, True)]:
            st = Stack(workers=w, executors=e, max_agg=m, mode=mode, barrier_elision=elide)
            try:
                seen.add(run(st, 8, 2)[1].checksum.hex())
            finally:
                st.close()
    assert seen == {want}


def test_seventeen_requests(stacks, golden):
    s = stacks(max_agg=8)
    agg = s.aggs[0]
    gate = threading.Event()
    # hold the device thread so everything queues behind the gate op
    s.device._work.put((agg.executor.queue, gate.wait, s.device._ids and
                        __import__("fake_device").FakeDevEvent()))
    agg.executor.queue._outstanding += 1
    srcs = [np.full(4, float(i)) for i in range(17)]
    dsts = [np.empty(4) for _ in range(17)]
    futs = [agg.schedule(0, srcs[i], dsts[i]) for i in range(17)]
    gate.set()
    when_all(futs, pool=s.runtime.pool).result(timeout=10)
    assert sorted(agg.batch_sizes) == [1, 8, 8]
    assert agg.reasons == {"full": 2, "idle": 1}
    assert [[v.hex() for v in d] for d in dsts] == golden["aggregation_17_m8"]["dst"]


def test_kind_errors(stacks):
    s = stacks()
    with pytest.raises(KindError):
        s.aggs[0].schedule("nope", np.ones(4), np.empty(4))
    with pytest.raises(KindError):
        s.aggs[0].register_kind("host", lambda v: None)
    with pytest.raises(StateError):
        s.aggs[0].first_slot_future(0)


def test_affine_kind_round_dependency(stacks):
    s = stacks(max_agg=8)
    agg = s.aggs[0]
    agg.register_kind("inc", affine_kernel(1.0, 1.0))

    def body():
        work, out = np.zeros(8), np.empty(8)
        for _ in range(5):
            yield agg.schedule("inc", work, out)
            work, out = out, work
        return work.copy()

    np.testing.assert_array_equal(s.runtime.submit(body).result(timeout=10), np.full(8, 5.0))


def test_criterion7_randomised_aggregation_soundness(stacks):
    rng = random.Random(20260815)
    s = stacks(workers=2, executors=4, max_agg=4)
    for _ in range(200):
        m = rng.randint(1, 16)
        n = rng.randint(1, 40)
        agg = AggregationExecutor(s.executors.acquire(), m, s.buffers, inject_barriers=False)
        for k in range(3):
            agg.register_kind(k, kernel_transform(k))
        srcs = [np.full(4, float(i)) for i in range(n)]
        dsts = [np.empty(4) for _ in range(n)]
        kinds = [rng.randrange(3) for _ in range(n)]
        futs = [agg.schedule(kinds[i], srcs[i], dsts[i]) for i in range(n)]
        when_all(futs, pool=s.runtime.pool).result(timeout=10)
        assert sum(agg.batch_sizes) == n and max(agg.batch_sizes) <= m
        for i in range(n):
            want = srcs[i].copy()
            mo.transform(want, kinds[i])
            np.testing.assert_array_equal(dsts[i], want)


@pytest.mark.parametrize("mode", [IntegrationMode.POLLING, IntegrationMode.HOSTTASK])
def test_nonblocking_modes_never_wait(stacks, mode):
    _, res = run(stacks(workers=4, executors=2, max_agg=4, mode=mode), 8, 2)
    assert sum(m.event_waits for m in res.per_step) == 0


def test_fence_waits(stacks):
    _, res = run(stacks(mode=IntegrationMode.FENCE, executors=2), 8, 1)
    assert res.per_step[0].event_waits > 0


def test_queue_future_rejects_out_of_order(stacks):
    s = stacks()

    class OOO:
        in_order = False

    with pytest.raises(OrderingError):
        s.integration.get_future_queue(OOO())


def test_bridged_event_counter(stacks):
    s = stacks()
    q = s.device.queue()
    before = s.integration.bridged_events
    s.integration.get_future(q.submit(make_dummy()))
    s.integration.get_future_queue(q)
    assert s.integration.bridged_events == before + 2


def test_device_gone_paths(stacks):
    s = stacks(mode=IntegrationMode.HOSTTASK)
    ex = s.executors.executors[0]
    s.device.destroy()
    ex.one_way(make_spin(1))
    f = ex.two_way(make_spin(1))
    assert f.status is FutureStatus.FAULTED and isinstance(f.error(), DeviceGoneError)


def test_buffer_pool_semantics():
    d = FakeDevice()
    try:
        pool = BufferPool(d)
        a = pool.alloc(256)
        pool.release(a)
        b = pool.alloc(256)
        assert b.id == a.id and pool.created == 1 and pool.reused == 1
        c = pool.alloc(128)
        assert c.id != a.id and pool.live_high_water == 2
        pool.release(b)
        with pytest.raises(PoolError):
            pool.release(b)
    finally:
        d.destroy()


def test_pool_round_robin(stacks):
    s4 = stacks(executors=4)
    assert [s4.executors.acquire().id for _ in range(8)] == [0, 1, 2, 3] * 2
    s = stacks(executors=128)
    counts = {}
    for _ in range(512):
        i = s.executors.acquire().id
        counts[i] = counts.get(i, 0) + 1
    assert len(counts) == 128 and set(counts.values()) == {4}


def test_min_tree_odd(runtime_factory):
    rt = runtime_factory(2)
    vals = [0.5, 0.125, 0.75, 0.25, 0.0625, 0.5, 1.5]
    ps = [make_promise(rt.pool) for _ in vals]
    fut = _min_tree([f for _, f in ps], rt.pool)
    for (p, _), v in zip(ps, vals):
        p.set_result(v)
    assert fut.result(timeout=10) == 0.0625


def test_buffer_reuse_across_steps(stacks):
    s = stacks(executors=1, max_agg=8)
    run(s, 8, 4)
    launches = sum(a.launches for a in s.aggs)
    assert s.buffers.created + s.buffers.reused == launches
    assert 0 < s.buffers.reused and s.buffers.created < launches


@pytest.mark.parametrize("block", [2, 3, 8, 16])
def test_coarsened_tasks_are_bit_identical(stacks, golden, block):
    s = stacks(workers=3, executors=2, max_agg=4)
    sc = build_scenario(ScenarioConfig(subgrids=16, steps=3, task_subgrids=block))
    by_grid = [s.aggs[i % len(s.aggs)] for i in range(16)]
    res = run_scenario(sc, s.runtime, s.device, s.aggs, by_grid)
    assert res.checksum.hex() == golden["machine"]["16x3"]["checksum"]
    cells = np.load(__import__("conftest").TESTS + "/golden/cells.npz")["cells_16x3"]
    np.testing.assert_array_equal(sc.cells(), cells)
    cs, dts = mo.run_reference(16, 3)
    assert res.dts == dts
