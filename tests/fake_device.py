"""CPU test double of the CUDA device duck type — TEST INFRASTRUCTURE ONLY.

Lets the CPU suite exercise the host logic of Integration / executors /
miniapp (futures, polling, aggregation, bit-exact goldens) without a GPU.
Ops execute in submission order on one background "device" thread; kernel
descriptors are applied with the oracle's numpy transform. The product
package never imports this (CudaDevice is the only product device).
"""

from __future__ import annotations

import itertools
import queue as _q
import threading
import time

import numpy as np

from oracle.miniapp_oracle import C1, C2
from paper_2303_08058_b200 import _native as N
from paper_2303_08058_b200.device import ClockMode, OpKind
from paper_2303_08058_b200.errors import DeviceGoneError
from paper_2303_08058_b200.runtime import _context


class FakeDevEvent:
    _ids = itertools.count()

    def __init__(self):
        self.id = next(FakeDevEvent._ids)
        self._done = threading.Event()
        self.completion_time = None

    def is_complete(self):
        return self._done.is_set()

    @property
    def status(self):
        from paper_2303_08058_b200.device import EventStatus
        return EventStatus.COMPLETE if self.is_complete() else EventStatus.SUBMITTED


class FakeBuffer:
    def __init__(self, buf_id, size_bytes):
        self.id = buf_id
        self.size_bytes = size_bytes
        self.host = np.zeros(size_bytes, dtype=np.uint8)
        self.dev = np.zeros(size_bytes, dtype=np.uint8)

    def f64(self):
        return self.host.view(np.float64)


def apply_kernel(kernel, view):
    if kernel.op == N.TB_OP_KIND:
        view *= C1[kernel.kind]
        view += C2[kernel.kind]
    elif kernel.op == N.TB_OP_AFFINE:
        view *= kernel.c1
        view += kernel.c2


class FakeQueue:
    def __init__(self, device, qid):
        self.device = device
        self.id = qid
        self._outstanding = 0
        self._lock = threading.Lock()

    in_order = True

    def submit(self, op):
        return self.device._submit(self, op)

    def incomplete_count(self):
        with self._lock:
            return self._outstanding


class FakeDevice:
    def __init__(self, op_delay=0.0, barrier_elision=False, hosttask_threads=2):
        self.clock_mode = ClockMode.REAL
        self.lazy_submit = False
        self.barrier_elision = barrier_elision
        self.op_delay = op_delay
        self.counters = dict(kernels=0, h2d=0, d2h=0, barriers=0, barriers_elided=0,
                             dummies=0, event_waits=0, hosttask_dispatched=0)
        self._lock = threading.Lock()
        self._alive = True
        self._work = _q.Queue()
        self._ids = itertools.count()
        self._queues = []
        self._host_tasks = {}
        self._thread = threading.Thread(target=self._run, name="fake-device", daemon=True)
        self._thread.start()
        self._ht_q = _q.Queue()
        self._ht_threads = [threading.Thread(target=self._ht_loop, name=f"tb-hosttask-{i}",
                                             daemon=True) for i in range(hosttask_threads)]
        for t in self._ht_threads:
            t.start()

    # duck type ----------------------------------------------------------
    def queue(self):
        q = FakeQueue(self, len(self._queues))
        self._queues.append(q)
        return q

    def alloc_buffer(self, n):
        return FakeBuffer(next(self._ids), n)

    def now(self):
        return time.perf_counter()

    def snapshot_counters(self):
        with self._lock:
            d = dict(self.counters)
        d["transfers"] = d["h2d"] + d["d2h"]
        return d

    def flush(self):
        pass

    def hosttask_thread_set(self):
        return set(self._ht_threads)

    def event_wait(self, ev):
        with self._lock:
            self.counters["event_waits"] += 1
        w = _context.current_worker()
        if w is not None:
            w.pool._note_blocked(1)
        try:
            while not ev._done.wait(0.005):
                if not self._alive:
                    raise DeviceGoneError("device destroyed while waiting")
        finally:
            if w is not None:
                w.pool._note_blocked(-1)

    def register_host_task(self, ev, cb, on_abandon=None):
        with self._lock:
            if not self._alive:
                raise DeviceGoneError("device destroyed")
            if ev.is_complete():
                self._ht_q.put((cb, on_abandon))
                return
            self._host_tasks.setdefault(ev.id, []).append((cb, on_abandon))

    def destroy(self):
        with self._lock:
            if not self._alive:
                return
            self._alive = False
            pending = [e for v in self._host_tasks.values() for e in v]
            self._host_tasks.clear()
        for _cb, ab in pending:
            if ab:
                ab(DeviceGoneError("device destroyed"))
        self._work.put(None)
        for _ in self._ht_threads:
            self._ht_q.put(None)

    def _count(self, key, n=1):
        with self._lock:
            self.counters[key] += n

    def _submit(self, queue, op):
        if not self._alive:
            raise DeviceGoneError("device destroyed")
        ev = FakeDevEvent()
        op.event = ev
        k = op.kind
        if k is OpKind.KERNEL:
            self._count("kernels")
            fn = None
            if op.buf is not None and op.kernel is not None:
                fn = lambda: apply_kernel(op.kernel, op.buf.f64()[:op.work_items])  # noqa: E731
            elif op.spin_ns:
                fn = lambda: time.sleep(op.spin_ns * 1e-9)  # noqa: E731
        elif k is OpKind.BARRIER:
            self._count("barriers_elided" if self.barrier_elision else "barriers")
            fn = None
        elif k is OpKind.DUMMY:
            self._count("dummies")
            fn = None
        else:
            self._count("h2d" if k is OpKind.COPY_H2D else "d2h")
            fn = None
        self._enqueue(queue, fn, ev)
        return ev

    def submit_batch(self, queue, kernel, staging, nbytes, barrier):
        if not self._alive:
            raise DeviceGoneError("device destroyed")
        self._count("h2d")
        self._count("kernels")
        self._count("d2h")
        if barrier:
            self._count("barriers_elided" if self.barrier_elision else "barriers")
        ev = FakeDevEvent()
        n = nbytes // 8

        def run():
            view = staging.f64()[:n].copy()
            apply_kernel(kernel, view)
            staging.f64()[:n] = view

        self._enqueue(queue, run, ev)
        return ev

    def _enqueue(self, queue, fn, ev):
        with queue._lock:
            queue._outstanding += 1
        self._work.put((queue, fn, ev))

    def _run(self):
        while True:
            item = self._work.get()
            if item is None:
                return
            queue, fn, ev = item
            if self.op_delay:
                time.sleep(self.op_delay)
            if fn is not None:
                fn()
            with queue._lock:
                queue._outstanding -= 1
            ev.completion_time = time.perf_counter()
            ev._done.set()
            with self._lock:
                tasks = self._host_tasks.pop(ev.id, [])
            for t in tasks:
                self._ht_q.put(t)

    def _ht_loop(self):
        while True:
            item = self._ht_q.get()
            if item is None:
                return
            cb, _ = item
            try:
                cb()
            except BaseException:
                pass
            self._count("hosttask_dispatched")
