"""Runtime host logic on CPU: futures, the work-stealing pool, the poll
registry's Python path (pkg/tests/test_futures.py, test_pool.py,
test_polling.py; acceptance criterion 6 part one)."""

import random
import statistics
import threading
import time
from time import perf_counter

import pytest

from conftest import FakeEvent
from paper_2303_08058_b200.errors import PromiseStateError, ShutdownError
from paper_2303_08058_b200.runtime import (EventCallback, FutureStatus, PollRegistry,
                                           Runtime, WorkerPool, blocked_region,
                                           future_then, make_promise,
                                           make_ready_future, when_all)


# ---------------------------------------------------------------- futures --
def test_continuation_runs_once_either_order():
    for attach_first in (True, False):
        p, f = make_promise()
        hits = []
        if attach_first:
            f.state.add_continuation(lambda: hits.append(1))
            p.set_result(3)
        else:
            p.set_result(3)
            f.state.add_continuation(lambda: hits.append(1))
        assert hits == [1] and f.value() == 3


def test_double_completion_raises():
    p, _ = make_promise()
    p.set_result(1)
    with pytest.raises(PromiseStateError):
        p.set_result(2)
    with pytest.raises(PromiseStateError):
        p.set_error(ValueError())


def test_value_of_pending_and_faulted():
    p, f = make_promise()
    with pytest.raises(RuntimeError):
        f.value()
    p.set_error(KeyError("x"))
    assert f.status is FutureStatus.FAULTED
    with pytest.raises(KeyError):
        f.value()
    with pytest.raises(TimeoutError):
        make_promise()[1].result(timeout=0.01)


def test_then_chain_order_and_fault_propagation(runtime_factory):
    rt = runtime_factory(2)
    p, f = make_promise(rt.pool)
    g = f.then(lambda v: v + 1).then(lambda v: v * 10)
    p.set_result(1)
    assert g.result(timeout=5) == 20
    p2, f2 = make_promise(rt.pool)
    called = []
    h = future_then(f2, lambda v: called.append(v), pool=rt.pool)
    p2.set_error(ValueError("boom"))
    with pytest.raises(ValueError):
        h.result(timeout=5)
    assert called == []
    bad = make_ready_future(1, pool=rt.pool).then(lambda v: 1 / 0)
    with pytest.raises(ZeroDivisionError):
        bad.result(timeout=5)


def test_when_all_order_empty_and_first_fault(runtime_factory):
    rt = runtime_factory(2)
    ps = [make_promise(rt.pool) for _ in range(5)]
    all_ = when_all([f for _, f in ps])
    for i in (3, 1, 4, 0, 2):
        ps[i][0].set_result(i * i)
    assert all_.result(timeout=5) == [0, 1, 4, 9, 16]
    assert when_all([]).result(timeout=1) == []
    ps = [make_promise(rt.pool) for _ in range(3)]
    w = when_all([f for _, f in ps])
    ps[1][0].set_error(KeyError("first"))
    ps[0][0].set_error(KeyError("second"))
    ps[2][0].set_result(0)
    with pytest.raises(KeyError, match="first"):
        w.result(timeout=5)


def test_randomised_attach_complete_race():
    rng = random.Random(5)
    for _ in range(200):
        p, f = make_promise()
        hits = []
        lock = threading.Lock()

        def attach():
            for _ in range(rng.randint(1, 5)):
                f.state.add_continuation(lambda: (lock.acquire(), hits.append(1),
                                                  lock.release()))

        t1 = threading.Thread(target=attach)
        t2 = threading.Thread(target=p.set_result)
        ts = [t1, t2] if rng.random() < 0.5 else [t2, t1]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        n_attached = len(hits)
        time.sleep(0)
        assert len(hits) == n_attached and f.is_ready()


# ------------------------------------------------------------------- pool --
def test_pool_runs_tasks_and_generators(runtime_factory):
    rt = runtime_factory(3)
    assert rt.submit(lambda: 41 + 1).result(timeout=5) == 42
    p, f = make_promise(rt.pool)

    def gen():
        v = yield f
        w = yield make_ready_future(5)
        return v + w

    out = rt.submit(gen)
    time.sleep(0.01)
    assert not out.is_ready()
    p.set_result(10)
    assert out.result(timeout=5) == 15


def test_suspension_frees_the_worker(runtime_factory):
    rt = runtime_factory(1)
    p, f = make_promise(rt.pool)

    def waiter():
        yield f
        return "resumed"

    w = rt.submit(waiter)
    other = rt.submit(lambda: "ran while suspended")
    assert other.result(timeout=5) == "ran while suspended"
    p.set_result(None)
    assert w.result(timeout=5) == "resumed"


def test_fault_thrown_into_generator(runtime_factory):
    rt = runtime_factory(2)
    p, f = make_promise(rt.pool)

    def gen():
        try:
            yield f
        except KeyError:
            return "caught"
        return "no"

    out = rt.submit(gen)
    p.set_error(KeyError("x"))
    assert out.result(timeout=5) == "caught"


def test_yielding_non_future_faults(runtime_factory):
    rt = runtime_factory(1)

    def gen():
        yield 3

    with pytest.raises(TypeError):
        rt.submit(gen).result(timeout=5)


def test_submit_after_shutdown_rejected():
    rt = Runtime(1)
    rt.shutdown()
    with pytest.raises(ShutdownError):
        rt.submit(lambda: 1)


def test_shutdown_faults_suspended_polling_entries():
    rt = Runtime(2)
    p, f = make_promise(rt.pool)
    rt.registry.add(EventCallback(FakeEvent(False), lambda: p.set_result(1),
                                  on_abandon=p.set_error))
    rt.shutdown()
    assert f.status is FutureStatus.FAULTED
    assert isinstance(f.error(), ShutdownError)


def test_worker_count_validation():
    with pytest.raises(ValueError):
        WorkerPool(0)


def test_many_tasks_from_foreign_threads(runtime_factory):
    rt = runtime_factory(4)
    futs, lock = [], threading.Lock()

    def producer(k):
        for i in range(250):
            f = rt.submit(lambda i=i, k=k: k * 1000 + i)
            with lock:
                futs.append(f)

    ts = [threading.Thread(target=producer, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    vals = sorted(f.result(timeout=10) for f in futs)
    assert vals == sorted(k * 1000 + i for k in range(4) for i in range(250))
    deadline = perf_counter() + 5
    while rt.pool.runnable_activity() and perf_counter() < deadline:
        time.sleep(1e-3)
    assert rt.pool.runnable_activity() == 0
    assert rt.pool.busy_seconds() > 0


def test_trace_records_labels():
    rt = Runtime(2, trace=True)
    try:
        rt.submit(lambda: None, label=("grid", 1)).result(timeout=5)
        deadline = perf_counter() + 2
        while not rt.pool.trace_log and perf_counter() < deadline:
            time.sleep(1e-3)
        assert rt.pool.trace_log[0][1] == ("grid", 1)
    finally:
        rt.shutdown()


def test_blocked_region_accounting(runtime_factory):
    rt = runtime_factory(1)
    seen = []

    def body():
        with blocked_region():
            seen.append(rt.pool.runnable_activity())
        return seen

    rt.submit(body).result(timeout=5)
    assert seen == [0]


# ----------------------------------------------------------- poll registry --
def test_exactly_once_and_pending_then_fire():
    reg = PollRegistry()
    ev = FakeEvent(False)
    hits = []
    reg.add(EventCallback(ev, lambda: hits.append(1)))
    assert reg.poll() == 0 and reg.pending_count() == 1
    ev.done = True
    assert reg.poll() == 1 and reg.poll() == 0
    assert hits == [1] and reg.fired_total == 1


def test_registration_order_preserved():
    reg = PollRegistry()
    evs = [FakeEvent(False) for _ in range(5)]
    order = []
    for i, e in enumerate(evs):
        reg.add(EventCallback(e, lambda i=i: order.append(i)))
    reg.poll()
    reg.add(EventCallback(FakeEvent(True), lambda: order.append("new")))
    for e in evs:
        e.done = True
    reg.poll()
    assert order == [0, 1, 2, 3, 4, "new"]


def test_producers_many_threads():
    reg = PollRegistry()
    lock, hits = threading.Lock(), [0]

    def cb():
        with lock:
            hits[0] += 1

    def producer():
        for _ in range(1000):
            reg.add(EventCallback(FakeEvent(True), cb))

    ts = [threading.Thread(target=producer) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    while reg.poll():
        pass
    assert hits[0] == 8000


def test_single_entrant_under_sixteen_hammer_threads():
    # acceptance criterion 6, part one (pkg/tests/test_acceptance.py:125-147)
    reg = PollRegistry()
    stop = threading.Event()

    def producer():
        while not stop.is_set():
            reg.add(EventCallback(FakeEvent(True), lambda: None))
            time.sleep(0)

    def hammer():
        while not stop.is_set():
            reg.poll()

    ts = [threading.Thread(target=producer)] + [threading.Thread(target=hammer)
                                                for _ in range(16)]
    for t in ts:
        t.start()
    time.sleep(0.5)
    stop.set()
    for t in ts:
        t.join()
    assert reg.entry_high_water == 1


def test_contended_poll_returns_immediately():
    reg = PollRegistry()
    reg._guard.acquire()
    try:
        samples = []
        for _ in range(500):
            t0 = perf_counter()
            assert reg.poll() == 0
            samples.append(perf_counter() - t0)
        assert statistics.median(samples) < 10e-6
    finally:
        reg._guard.release()


def test_callback_fault_isolated():
    reg = PollRegistry()
    hits = []
    reg.add(EventCallback(FakeEvent(True), lambda: 1 / 0))
    reg.add(EventCallback(FakeEvent(True), lambda: hits.append(1)))
    assert reg.poll() == 2 and hits == [1]


def test_abandon_all_runs_complete_and_abandons_rest():
    reg = PollRegistry()
    hits, errs = [], []
    reg.add(EventCallback(FakeEvent(True), lambda: hits.append(1), errs.append))
    reg.add(EventCallback(FakeEvent(False), lambda: hits.append(2), errs.append))
    assert reg.abandon_all(ShutdownError("x")) == 1
    assert hits == [1] and len(errs) == 1 and not reg.has_waiting()


def test_flush_hook_runs_each_poll():
    reg = PollRegistry()
    calls = []
    reg.add_flush_hook(lambda: calls.append(1))
    reg.poll()
    reg.poll()
    assert calls == [1, 1]


def test_idle_workers_poll_the_registry(runtime_factory):
    rt = runtime_factory(2)
    ev = FakeEvent(False)
    p, f = make_promise(rt.pool)
    rt.registry.add(EventCallback(ev, lambda: p.set_result("fired")))
    time.sleep(0.01)
    assert not f.is_ready()
    ev.done = True
    assert f.result(timeout=5) == "fired"
