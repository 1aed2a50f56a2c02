"""The reference-facing machine (runtime + bridge + aggregation executors +
mini-app) on the CUDA device: goldens in every integration mode, counts,
aggregation semantics, fault paths (pkg/tests/test_miniapp.py,
test_executors.py, test_bridge.py, test_acceptance.py criteria 1, 2, 6)."""

import threading
import time

import numpy as np
import pytest

from conftest import fx
from oracle import miniapp_oracle as mo

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2303_08058_b200 import (AggregationExecutor, BufferPool, CudaDevice,  # noqa: E402
                                   DeviceGoneError, ExecutorPool, FutureStatus,
                                   Integration, IntegrationMode, KindError, Runtime,
                                   ScenarioConfig, ShutdownError, StateError,
                                   affine_kernel, build_scenario, kernel_transform,
                                   make_dummy, make_kernel, make_spin, run_scenario,
                                   when_all)

MODES = [IntegrationMode.POLLING, IntegrationMode.HOSTTASK, IntegrationMode.FENCE]


class Stack:
    def __init__(self, workers=2, mode=IntegrationMode.POLLING, executors=1, max_agg=4,
                 inject_barriers=True, barrier_elision=False, register=True,
                 record_timeline=False):
        self.runtime = Runtime(workers, seed=7)
        self.device = CudaDevice(barrier_elision=barrier_elision,
                                 record_timeline=record_timeline)
        self.integration = Integration(self.runtime, self.device, mode)
        self.executors = ExecutorPool(self.integration, executors)
        self.buffers = BufferPool(self.device)
        self.aggs = [AggregationExecutor(ex, max_agg, self.buffers,
                                         inject_barriers=inject_barriers)
                     for ex in self.executors.executors]
        if register:
            for a in self.aggs:
                for k in range(5):
                    a.register_kind(k, kernel_transform(k))

    def drive(self, fut, timeout=60.0):
        return fut.result(timeout=timeout)

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
        try:
            s.close()
        except Exception:
            pass


def run(stack, subgrids, steps):
    sc = build_scenario(ScenarioConfig(subgrids=subgrids, steps=steps))
    by_grid = [stack.aggs[i % len(stack.aggs)] for i in range(subgrids)]
    return sc, run_scenario(sc, stack.runtime, stack.device, stack.aggs, by_grid,
                            engine="python")


@pytest.mark.parametrize("mode", MODES)
def test_machine_goldens_every_mode(stacks, golden, mode):
    lit = golden["reference_test_literals"]
    s = stacks(workers=2, executors=2, max_agg=8, mode=mode)
    _, res = run(s, 4, 2)
    assert res.checksum == fx(lit["GOLDEN_4X2"])
    assert res.dts == [fx(h) for h in lit["GOLDEN_4X2_DTS"]]
    s2 = stacks(workers=4, executors=3, max_agg=4, mode=mode)
    sc, res = run(s2, 16, 3)
    assert res.checksum.hex() == golden["machine"]["16x3"]["checksum"]
    cells = np.load(__import__("conftest").TESTS + "/golden/cells.npz")["cells_16x3"]
    np.testing.assert_array_equal(sc.cells(), cells)


def test_unfused_counts_exact(stacks, golden):
    # pkg/tests/test_miniapp.py:65-75
    s = stacks(executors=1, max_agg=1)
    _, res = run(s, 8, 2)
    for m in res.per_step:
        assert m.launches == 8 * 15
        assert m.transfers == 8 * 30
        assert sum(m.batch_sizes) == 120
        assert m.reasons_full == 120 and m.reasons_idle == 0
        assert m.event_waits == 0
    assert res.checksum == fx(golden["reference_test_literals"]["GOLDEN_8X2"])


def test_criterion1_counts_512(stacks, golden):
    s = stacks(workers=8, executors=32, max_agg=1)
    _, res = run(s, 512, 1)
    m = res.per_step[0]
    want = golden["machine_counts_512x1_m1"]
    assert m.launches == want["kernels"] == 7680
    assert m.transfers == want["transfers"] == 15360
    assert res.checksum.hex() == want["checksum"]


def test_fused_run_batches_and_matches(stacks, golden):
    s = stacks(executors=1, max_agg=4)
    _, res = run(s, 8, 2)
    assert sum(sz for m in res.per_step for sz in m.batch_sizes) == 8 * 15 * 2
    assert res.checksum == fx(golden["reference_test_literals"]["GOLDEN_8X2"])


def test_self_ring(stacks):
    s = stacks(executors=1, max_agg=2)
    _, res = run(s, 1, 2)
    cs, dts = mo.run_reference(1, 2)
    assert res.checksum == cs and res.dts == dts


@pytest.mark.parametrize("mode", MODES)
def test_criterion2_checksum_invariant(golden, mode):
    want = golden["reference_test_literals"]["GOLDEN_8X2"]
    seen = set()
    for e, m, w, elide in [(1, 1, 1, False), (8, 8, 4, True), (32, 32, 8, False),
                           (8, 1, 8, True), (1, 32, 4, False)]:
        st = Stack(workers=w, executors=e, max_agg=m, mode=mode, barrier_elision=elide)
        try:
            _, res = run(st, 8, 2)
            seen.add(res.checksum.hex())
        finally:
            st.close()
    assert seen == {fx(want).hex()}


def test_seventeen_requests_partition(stacks, golden):
    s = stacks(max_agg=8)
    agg = s.aggs[0]
    agg.executor.one_way(make_spin(20_000))     # keep the queue busy 20 ms
    srcs = [np.full(4, float(i)) for i in range(17)]
    dsts = [np.empty(4) for _ in range(17)]
    futs = [agg.schedule(0, srcs[i], dsts[i]) for i in range(17)]
    s.drive(when_all(futs, pool=s.runtime.pool))
    assert sorted(agg.batch_sizes) == [1, 8, 8]
    assert agg.reasons == {"full": 2, "idle": 1}
    g = golden["aggregation_17_m8"]
    assert [[v.hex() for v in d] for d in dsts] == g["dst"]


def test_lone_request_launches_on_idle(stacks):
    s = stacks(max_agg=2)
    agg = s.aggs[0]
    src = np.arange(4, dtype=np.float64)
    dst = np.empty(4)
    s.drive(agg.schedule(1, src, dst))
    assert agg.batch_sizes == [1] and agg.reasons == {"full": 0, "idle": 1}
    want = src.copy()
    mo.transform(want, 1)
    np.testing.assert_array_equal(dst, want)


def test_first_slot_future_one_probe_per_batch(stacks):
    s = stacks(max_agg=4)
    agg = s.aggs[0]
    agg.executor.one_way(make_spin(20_000))
    with pytest.raises(StateError):
        agg.first_slot_future(0)
    before = s.integration.bridged_events
    f1 = agg.schedule(0, np.ones(4), np.empty(4))
    probe = agg.first_slot_future(0)
    assert s.integration.bridged_events == before + 1
    f2 = agg.schedule(0, np.ones(4), np.empty(4))
    assert agg.first_slot_future(0) is probe
    s.drive(when_all([f1, f2], pool=s.runtime.pool))
    assert agg.reasons["idle"] == 1


def test_mixed_kinds_never_co_batch(stacks):
    s = stacks(max_agg=8)
    agg = s.aggs[0]
    agg.executor.one_way(make_spin(20_000))
    dsts = [np.empty(4) for _ in range(6)]
    futs = [agg.schedule(i % 3, np.full(4, float(i)), dsts[i]) for i in range(6)]
    s.drive(when_all(futs, pool=s.runtime.pool))
    assert sorted(agg.batch_sizes) == [2, 2, 2]


def test_round_dependency_with_affine_kind(stacks):
    s = stacks(max_agg=8)
    agg = s.aggs[0]
    agg.register_kind("inc", affine_kernel(1.0, 1.0))
    with pytest.raises(KindError):
        agg.register_kind("host", lambda v: v.__iadd__(1.0))

    def body():
        work, out = np.zeros(8), np.empty(8)
        for _ in range(5):
            yield agg.schedule("inc", work, out)
            work, out = out, work
        return work.copy()

    np.testing.assert_array_equal(s.drive(s.runtime.submit(body)), np.full(8, 5.0))


@pytest.mark.parametrize("mode", [IntegrationMode.POLLING, IntegrationMode.HOSTTASK])
def test_nonblocking_modes_never_wait(stacks, mode):
    s = stacks(workers=4, executors=2, max_agg=4, mode=mode)
    _, res = run(s, 8, 2)
    assert sum(m.event_waits for m in res.per_step) == 0


def test_fence_mode_waits(stacks):
    s = stacks(workers=2, executors=2, max_agg=4, mode=IntegrationMode.FENCE)
    _, res = run(s, 8, 1)
    assert res.per_step[0].event_waits > 0


def test_polling_ready_within_one_poll_after_completion(stacks):
    s = stacks()
    q = s.device.queue()
    ev = q.submit(make_kernel(16))
    s.device.synchronize()
    fut = s.integration.get_future_polling(ev)
    polls = 0
    while not fut.is_ready() and polls < 50:
        s.runtime.registry.poll()
        polls += 1
    assert fut.is_ready() and polls <= 1


def test_hosttask_sets_future_on_device_thread(stacks):
    s = stacks(mode=IntegrationMode.HOSTTASK)
    q = s.device.queue()
    q.submit(make_spin(2_000))
    ev = q.submit(make_kernel(16))
    fut = s.integration.get_future(ev)
    who, done = [], threading.Event()
    fut.state.add_continuation(lambda: (who.append(threading.current_thread()), done.set()))
    assert done.wait(10.0)
    assert who[0] in s.device.hosttask_thread_set()
    assert who[0] not in s.runtime.pool.worker_threads()


def test_hosttask_thousand_events_exactly_once(stacks):
    s = stacks(mode=IntegrationMode.HOSTTASK, executors=8)
    queues = [ex.queue for ex in s.executors.executors]
    lock, fired = threading.Lock(), [0]

    def bump():
        with lock:
            fired[0] += 1

    futs = []
    for i in range(1000):
        f = s.integration.get_future(queues[i % 8].submit(make_dummy()))
        f.state.add_continuation(bump)
        futs.append(f)
    deadline = time.perf_counter() + 20
    while fired[0] < 1000 and time.perf_counter() < deadline:
        time.sleep(1e-3)
    assert fired[0] == 1000 and all(f.is_ready() for f in futs)


def test_fence_blocks_for_the_op():
    rt = Runtime(1)
    d = CudaDevice()
    try:
        integ = Integration(rt, d, IntegrationMode.FENCE)
        q = d.queue()
        ev = q.submit(make_spin(20_000))
        t0 = time.perf_counter()
        fut = integ.get_future(ev)
        el = time.perf_counter() - t0
        assert fut.is_ready() and ev.is_complete()
        assert el >= 0.015
        assert d.snapshot_counters()["event_waits"] == 1
    finally:
        rt.shutdown()
        d.destroy()


def test_queue_future_dominates_prior_ops(stacks):
    s = stacks()
    q = s.device.queue()
    evs = [q.submit(make_spin(2_000)) for _ in range(5)]
    fut = s.integration.get_future_queue(q)
    s.drive(fut)
    assert all(e.is_complete() for e in evs)


def test_successive_queue_futures_ordered(stacks):
    s = stacks()
    q = s.device.queue()
    q.submit(make_spin(5_000))
    f1 = s.integration.get_future_queue(q)
    f2 = s.integration.get_future_queue(q)
    seen = []
    f1.state.add_continuation(lambda: seen.append("first"))
    f2.state.add_continuation(lambda: seen.append("second"))
    s.drive(f2)
    time.sleep(0.01)
    assert seen == ["first", "second"]


def test_shutdown_faults_pending_polling_bridge():
    rt = Runtime(2)
    d = CudaDevice()
    try:
        integ = Integration(rt, d, IntegrationMode.POLLING)
        q = d.queue()
        ev = q.submit(make_spin(300_000))
        fut = integ.get_future(ev)
        rt.shutdown(timeout=1.0)
        assert fut.status is FutureStatus.FAULTED
        assert isinstance(fut.error(), ShutdownError)
    finally:
        d.destroy()


def test_destroy_faults_pending_hosttask_bridge():
    rt = Runtime(2)
    d = CudaDevice()
    try:
        integ = Integration(rt, d, IntegrationMode.HOSTTASK)
        q = d.queue()
        ev = q.submit(make_spin(300_000))
        fut = integ.get_future(ev)
        d.destroy()
        assert fut.status is FutureStatus.FAULTED
        assert isinstance(fut.error(), DeviceGoneError)
    finally:
        rt.shutdown()


def test_executor_ops_after_destroy(stacks):
    s = stacks()
    ex = s.executors.executors[0]
    s.device.destroy()
    ex.one_way(make_kernel(4))
    fut = ex.two_way(make_kernel(4))
    assert fut.status is FutureStatus.FAULTED
    assert isinstance(fut.error(), DeviceGoneError)


def test_native_poll_registry_single_entrant_under_hammer(stacks):
    s = stacks()
    reg = s.runtime.registry
    q = s.device.queue()
    stop = threading.Event()
    fired = [0]
    lock = threading.Lock()

    def cb():
        with lock:
            fired[0] += 1

    from paper_2303_08058_b200 import EventCallback

    def producer():
        for _ in range(2000):
            reg.add(EventCallback(q.submit(make_dummy()), cb))

    def hammer():
        while not stop.is_set():
            reg.poll()

    ts = [threading.Thread(target=hammer) for _ in range(16)]
    for t in ts:
        t.start()
    producer()
    deadline = time.perf_counter() + 20
    while fired[0] < 2000 and time.perf_counter() < deadline:
        time.sleep(1e-3)
    stop.set()
    for t in ts:
        t.join()
    assert fired[0] == 2000
    assert reg.entry_high_water == 1


def test_lazy_device_flushes_from_the_poll_hook():
    # pkg/tests/test_bridge.py:234-251 on CUDA: parked until a poll flushes
    rt = Runtime(2)
    d = CudaDevice(lazy_submit=True)
    try:
        integ = Integration(rt, d, IntegrationMode.POLLING)
        q = d.queue()
        ev = q.submit(make_kernel(16))
        assert d.held_count() == 1 and d.snapshot_counters()["kernels"] == 0
        assert not ev.is_complete()
        fut = integ.get_future(ev)
        fut.result(timeout=10)               # idle workers poll -> flush hook
        assert ev.is_complete() and d.held_count() == 0
        assert d.snapshot_counters()["kernels"] == 1
    finally:
        rt.shutdown()
        d.destroy()


@pytest.mark.parametrize("mode", MODES)
def test_lazy_device_machine_golden(golden, mode):
    rt = Runtime(2, seed=3)
    d = CudaDevice(lazy_submit=True)
    try:
        integ = Integration(rt, d, mode)
        pool = ExecutorPool(integ, 2)
        bufs = BufferPool(d)
        aggs = [AggregationExecutor(ex, 4, bufs) for ex in pool.executors]
        for a in aggs:
            for k in range(5):
                a.register_kind(k, kernel_transform(k))
        sc = build_scenario(ScenarioConfig(subgrids=8, steps=2))
        res = run_scenario(sc, rt, d, aggs, [aggs[i % 2] for i in range(8)], engine="python")
        assert res.checksum == fx(golden["reference_test_literals"]["GOLDEN_8X2"])
    finally:
        rt.shutdown()
        d.destroy()


def test_record_timeline_rows_per_op():
    # VirtualDevice(record_timeline=True) rows (src/device.py:223-224,512-514)
    # from CUDA timing events around every op
    from paper_2303_08058_b200.device import make_barrier, make_dummy, make_spin
    d = CudaDevice(0, record_timeline=True)
    try:
        q0, q1 = d.queue(), d.queue()
        script = [(q0, make_spin(300)), (q1, make_spin(100)), (q0, make_barrier()),
                  (q1, make_dummy()), (q0, make_spin(50)), (q1, make_spin(200))]
        for q, op in script:
            q.submit(op)
        d.synchronize()
        rows = d.timeline
        assert len(rows) == len(script)
        by_q = {}
        for qid, idx, kind, start, end in rows:
            assert 0.0 <= start <= end
            by_q.setdefault(qid, []).append((idx, kind, start, end))
        for qid, ops in by_q.items():
            ops.sort()
            assert [o[0] for o in ops] == list(range(len(ops)))
            for a, b in zip(ops, ops[1:]):           # in-order queues
                assert b[2] >= a[3] - 1e-6
        spins = [r for r in rows if r[0] == q0.id and r[2] == "kernel"]
        assert spins[0][4] - spins[0][3] >= 290e-6    # the 300 us spin
        assert [r[2] for r in sorted(rows) if r[0] == q0.id] == ["kernel", "barrier", "kernel"]
    finally:
        d.destroy()


def test_record_timeline_through_aggregation(stacks):
    s = stacks(executors=1, max_agg=4, record_timeline=True)
    src = np.linspace(0.0, 1.0, 512)
    futs = [s.aggs[0].schedule(0, src, np.empty(512)) for _ in range(3)]
    for f in futs:
        f.result(timeout=30)
    s.device.synchronize()
    kinds = [r[2] for r in sorted(s.device.timeline)]
    # the batch's ops, one row each, plus the idleness probe's marker
    assert kinds.count("h2d") == kinds.count("d2h") == kinds.count("barrier") >= 1
    assert kinds.count("dummy") >= 1
