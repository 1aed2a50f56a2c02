"""Virtual-clock CPU double of the device duck type — TEST INFRASTRUCTURE ONLY.

Keeps the reference's acceptance criteria 8 (byte-identical virtual runs,
pkg/tests/test_acceptance.py:190-202) and 9 (two-queue timeline equals an
independent simulator, pkg/tests/test_acceptance.py:204-241) testable without
a GPU. The product device is CudaDevice (real clock
only); the reference's own virtual clock lives at src/device.py:322-343 and
its pump at src/pump.py:30-78 — this is a separate, from-scratch double of the
same documented semantics:

* time is a float that moves only when the pump calls ``advance_to_next()``;
* each queue is in order: its head starts when the previous op completed and,
  if it is a kernel, a device-wide compute slot is free (``compute_slots``);
* a kernel that finds every slot taken parks; freed slots go first to the
  queue that freed one (it re-kicks its own next op), then to parked queues
  by (time parked, queue id);
* op durations follow the latency model (src/device.py:63-81 defaults);
* completions due at the same instant are processed in start order;
* barrier elision: an elided barrier's event rides on the queue's newest op;
* kernel descriptors transform their buffer with the oracle's numpy
  arithmetic when the op starts (the reference runs closures at op start);
* host tasks run on ``tb-hosttask-i`` threads; fence waits block the calling
  worker (counted as blocked in the pool) until the pump completes the op.

``VirtualClockPump`` advances the clock only when the host side is
quiescent (no progressable pool activity, no queued or running host task, no
fence waiter whose op already completed), so every burst of host work happens
at one virtual instant and the whole run is reproducible.
"""

from __future__ import annotations

import heapq
import itertools
import threading
import time
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional

from fake_device import FakeBuffer, apply_kernel
from paper_2303_08058_b200.device import ClockMode, EventStatus, OpKind
from paper_2303_08058_b200.errors import DeviceGoneError, ModeError
from paper_2303_08058_b200.runtime import _context


@dataclass(frozen=True)
class Latency:
    """Op durations in seconds (defaults: src/device.py:63-72)."""
    kernel_fixed: float = 50e-6
    kernel_per_item: float = 0.05e-6
    copy_per_byte: float = 0.2e-9
    barrier_cost: float = 10e-6

    def of(self, kind: OpKind, items: int, nbytes: int) -> float:
        if kind is OpKind.KERNEL:
            return self.kernel_fixed + self.kernel_per_item * items
        if kind in (OpKind.COPY_H2D, OpKind.COPY_D2H):
            return self.copy_per_byte * nbytes
        if kind is OpKind.BARRIER:
            return self.barrier_cost
        return self.kernel_fixed          # DUMMY queue marker


class VEvent:
    _ids = itertools.count()

    def __init__(self):
        self.id = next(VEvent._ids)
        self._status = EventStatus.SUBMITTED
        self.completion_time: Optional[float] = None
        self.riders: List["VEvent"] = []      # elided barriers completing with it

    def is_complete(self) -> bool:
        return self._status is EventStatus.COMPLETE

    @property
    def status(self) -> EventStatus:
        return self._status


class _VOp:
    __slots__ = ("queue", "index", "kind", "items", "nbytes", "run", "event", "start", "end",
                 "seq")

    def __init__(self, queue, index, kind, items, nbytes, run, event):
        self.queue, self.index, self.kind = queue, index, kind
        self.items, self.nbytes, self.run, self.event = items, nbytes, run, event
        self.start = self.end = None
        self.seq = -1


class VQueue:
    in_order = True

    def __init__(self, device: "VirtualClockDevice", qid: int):
        self.device = device
        self.id = qid
        self.backlog: List[_VOp] = []
        self.active: Optional[_VOp] = None
        self.submitted = 0
        self.newest: Optional[VEvent] = None

    def submit(self, op) -> VEvent:
        return self.device._submit(self, op)

    def incomplete_count(self) -> int:
        with self.device._lock:
            return len(self.backlog) + (1 if self.active is not None else 0)


class VirtualClockDevice:
    """The device duck type (CudaDevice / the reference's VirtualDevice) on a
    discrete-event virtual clock."""

    def __init__(self, compute_slots: int = 16, latency: Optional[Latency] = None,
                 barrier_elision: bool = False, record_timeline: bool = False,
                 hosttask_threads: int = 2, clock_mode: ClockMode = ClockMode.VIRTUAL,
                 **_ignored):
        if clock_mode is not ClockMode.VIRTUAL:
            raise ModeError("VirtualClockDevice runs on the virtual clock only")
        if compute_slots < 1:
            raise ValueError("compute_slots must be >= 1")
        self.clock_mode = ClockMode.VIRTUAL
        self.lazy_submit = False
        self.compute_slots = compute_slots
        self.latency = latency or Latency()
        self.barrier_elision = barrier_elision
        self.record_timeline = record_timeline
        self.timeline: list = []
        self.counters = dict(kernels=0, h2d=0, d2h=0, barriers=0, barriers_elided=0,
                             dummies=0, event_waits=0, hosttask_dispatched=0)
        self._lock = threading.Lock()
        self._wake = threading.Condition(self._lock)
        self._alive = True
        self._now = 0.0
        self._queues: List[VQueue] = []
        self._running: list = []            # heap of (end, seq, op)
        self._slots_used = 0
        self._parked: list = []             # [(time parked, queue id, queue)]
        self._seq = itertools.count()
        self._buf_ids = itertools.count()
        self._host_tasks: Dict[int, list] = {}
        self._waiters: Dict[VEvent, int] = {}
        self._ht_items: list = []           # queued host-task callbacks
        self._ht_busy = 0                   # callbacks running
        self._ht_closed = False
        self._ht_lock = threading.Lock()
        self._ht_cv = threading.Condition(self._ht_lock)
        self._ht_threads = [threading.Thread(target=self._ht_loop, name=f"tb-hosttask-{i}",
                                             daemon=True) for i in range(hosttask_threads)]
        for t in self._ht_threads:
            t.start()

    # ------------------------------------------------------------ duck type
    def queue(self) -> VQueue:
        with self._lock:
            q = VQueue(self, len(self._queues))
            self._queues.append(q)
            return q

    def alloc_buffer(self, nbytes: int):
        return FakeBuffer(next(self._buf_ids), nbytes)

    def now(self) -> float:
        return self._now

    def flush(self) -> None:
        pass

    def hosttask_thread_set(self) -> set:
        return set(self._ht_threads)

    def snapshot_counters(self) -> dict:
        with self._lock:
            d = dict(self.counters)
        d["transfers"] = d["h2d"] + d["d2h"]
        return d

    def event_status(self, ev: VEvent) -> EventStatus:
        return ev.status

    def has_pending(self) -> bool:
        with self._lock:
            return bool(self._running)

    def hosttask_backlog(self) -> int:
        with self._ht_lock:
            return len(self._ht_items) + self._ht_busy

    def event_wait(self, ev: VEvent) -> None:
        """FENCE: block the calling worker until the pump completes ``ev``."""
        w = _context.current_worker()
        pool = w.pool if w is not None else None
        with self._lock:
            self.counters["event_waits"] += 1
            if not self._alive:
                raise DeviceGoneError("device destroyed")
            if ev.is_complete():
                return
            if pool is not None:
                pool._note_blocked(+1)
            self._waiters[ev] = self._waiters.get(ev, 0) + 1
            try:
                while not ev.is_complete():
                    if not self._alive:
                        raise DeviceGoneError("device destroyed while waiting")
                    self._wake.wait(0.05)
            finally:
                # leave the blocked count and the waiter table together, so
                # the pump never advances between this wake-up and the resume
                n = self._waiters[ev] - 1
                if n:
                    self._waiters[ev] = n
                else:
                    del self._waiters[ev]
                if pool is not None:
                    pool._note_blocked(-1)

    def register_host_task(self, ev: VEvent, cb: Callable[[], None],
                           on_abandon: Optional[Callable] = None) -> None:
        with self._lock:
            if not self._alive:
                raise DeviceGoneError("device destroyed")
            if ev.is_complete():
                self._ht_put(cb, on_abandon)
                return
            self._host_tasks.setdefault(ev.id, []).append((cb, on_abandon))

    def submit_batch(self, queue: VQueue, kernel, staging, nbytes: int, barrier: bool):
        """The reference's four ops of one aggregated launch
        (src/executors.py:277-284): H2D ; KERNEL ; [BARRIER] ; D2H."""
        from paper_2303_08058_b200.device import DeviceOp
        n = nbytes // 8
        self._submit(queue, DeviceOp(OpKind.COPY_H2D, nbytes=nbytes))
        self._submit(queue, DeviceOp(OpKind.KERNEL, work_items=n, kernel=kernel, buf=staging))
        if barrier:
            self._submit(queue, DeviceOp(OpKind.BARRIER))
        return self._submit(queue, DeviceOp(OpKind.COPY_D2H, nbytes=nbytes))

    def destroy(self) -> None:
        with self._lock:
            if not self._alive:
                return
            self._alive = False
            pending = [e for v in self._host_tasks.values() for e in v]
            self._host_tasks.clear()
            self._wake.notify_all()
        for _cb, ab in pending:
            if ab is not None:
                try:
                    ab(DeviceGoneError("device destroyed"))
                except BaseException:  # noqa: BLE001
                    pass
        with self._ht_cv:
            self._ht_closed = True
            self._ht_cv.notify_all()
        for t in self._ht_threads:
            t.join(timeout=2.0)

    # ------------------------------------------------------------- the clock
    def advance_to_next(self) -> bool:
        """Move the clock to the earliest running op's completion and process
        every completion due then; False when nothing is running."""
        with self._lock:
            if not self._running:
                return False
            t = self._running[0][0]
            self._now = max(self._now, t)
            while self._running and self._running[0][0] <= t:
                _, _, op = heapq.heappop(self._running)
                self._complete(op, t)
            self._wake.notify_all()
            return True

    def safe_to_advance(self, progressable: Callable[[], int]) -> bool:
        with self._lock:
            if any(n > 0 and ev.is_complete() for ev, n in self._waiters.items()):
                return False
        if self.hosttask_backlog():
            return False
        return progressable() == 0

    # ------------------------------------------------------------ internals
    def _submit(self, queue: VQueue, op) -> VEvent:
        with self._lock:
            if not self._alive:
                raise DeviceGoneError("device destroyed")
            ev = VEvent()
            op.event = ev
            op.queue = queue
            op.index = queue.submitted
            queue.submitted += 1
            kind = op.kind
            key = {OpKind.KERNEL: "kernels", OpKind.COPY_H2D: "h2d",
                   OpKind.COPY_D2H: "d2h", OpKind.DUMMY: "dummies"}.get(kind)
            if kind is OpKind.BARRIER:
                if self.barrier_elision:
                    self.counters["barriers_elided"] += 1
                    tail = queue.newest
                    if tail is None or tail.is_complete():
                        ev._status = EventStatus.COMPLETE
                        ev.completion_time = self._now
                    else:
                        tail.riders.append(ev)
                    return ev
                key = "barriers"
            self.counters[key] += 1
            run = None
            if kind is OpKind.KERNEL and op.kernel is not None and op.buf is not None:
                run = (op.kernel, op.buf, op.work_items)
            vop = _VOp(queue, op.index, kind, op.work_items, op.nbytes, run, ev)
            queue.backlog.append(vop)
            queue.newest = ev
            self._kick(queue, self._now)
            return ev

    def _kick(self, queue: VQueue, t: float) -> None:
        if queue.active is not None or not queue.backlog:
            return
        head = queue.backlog[0]
        if head.kind is OpKind.KERNEL and self._slots_used >= self.compute_slots:
            if all(p[2] is not queue for p in self._parked):
                self._parked.append((t, queue.id, queue))
            return
        self._start(queue, t)

    def _start(self, queue: VQueue, t: float) -> None:
        op = queue.backlog.pop(0)
        op.start = t
        op.end = t + self.latency.of(op.kind, op.items, op.nbytes)
        op.seq = next(self._seq)
        op.event._status = EventStatus.RUNNING
        queue.active = op
        if op.kind is OpKind.KERNEL:
            self._slots_used += 1
        if op.run is not None:
            kernel, buf, n = op.run
            view = buf.f64()[:n]
            work = view.copy()
            apply_kernel(kernel, work)
            view[:] = work
        heapq.heappush(self._running, (op.end, op.seq, op))

    def _complete(self, op: _VOp, t: float) -> None:
        queue = op.queue
        queue.active = None
        if op.kind is OpKind.KERNEL:
            self._slots_used -= 1
        if self.record_timeline:
            self.timeline.append((queue.id, op.index, op.kind.value, op.start, t))
        for ev in [op.event] + op.event.riders:
            ev._status = EventStatus.COMPLETE
            ev.completion_time = t
            for cb, ab in self._host_tasks.pop(ev.id, []):
                self._ht_put(cb, ab)
        # the freed queue first, then parked queues by (time parked, id)
        self._kick(queue, t)
        self._parked.sort(key=lambda p: (p[0], p[1]))
        while self._parked and self._slots_used < self.compute_slots:
            _, _, q = self._parked.pop(0)
            if q.active is None and q.backlog:
                self._start(q, t)

    def _ht_put(self, cb, ab) -> None:
        with self._ht_cv:
            self._ht_items.append((cb, ab))
            self._ht_cv.notify()

    def _ht_loop(self) -> None:
        while True:
            with self._ht_cv:      # take an item and count it busy atomically
                while not self._ht_items and not self._ht_closed:
                    self._ht_cv.wait()
                if not self._ht_items:
                    return
                item = self._ht_items.pop(0)
                self._ht_busy += 1
            try:
                item[0]()
            except BaseException:  # noqa: BLE001 - callback faults land in futures
                pass
            finally:
                with self._lock:
                    self.counters["hosttask_dispatched"] += 1
                with self._ht_lock:
                    self._ht_busy -= 1


class VirtualClockPump:
    """Drives a future to completion on a VirtualClockDevice: poll the
    runtime's registry, let runnable host work run, and advance the clock
    only at host quiescence."""

    def __init__(self, runtime, device: VirtualClockDevice, watchdog_seconds: float = 120.0):
        if device.clock_mode is not ClockMode.VIRTUAL:
            raise ModeError("the pump needs a virtual-clock device")
        self.runtime = runtime
        self.device = device
        self.watchdog_seconds = watchdog_seconds

    def drive(self, fut):
        registry = self.runtime.registry
        pool = self.runtime.pool
        dev = self.device
        deadline = time.monotonic() + self.watchdog_seconds
        idle_rounds = 0
        while not fut.is_ready():
            if time.monotonic() > deadline:
                raise TimeoutError(
                    f"virtual pump watchdog: progressable={pool.progressable_activity()} "
                    f"registry={registry.pending_count()} hosttasks={dev.hosttask_backlog()}")
            if registry.poll():
                idle_rounds = 0
                continue
            if not dev.safe_to_advance(pool.progressable_activity):
                time.sleep(2e-6)
                idle_rounds = 0
                continue
            if dev.advance_to_next():
                idle_rounds = 0
                continue
            idle_rounds += 1
            if idle_rounds > 20000:
                raise RuntimeError("virtual pump stuck: quiescent, nothing to advance, "
                                   "future not ready")
            time.sleep(10e-6)
        return fut.result(timeout=0)


def make_virtual_stack(**device_kw):
    """(device factory, pump factory) for the CLI's injectable devices."""
    return (lambda **kw: VirtualClockDevice(**{**kw, **device_kw}),
            lambda runtime, device, watchdog: VirtualClockPump(runtime, device, watchdog))

