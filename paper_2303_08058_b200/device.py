"""CUDA device layer: the B200 replacement for the reference's simulated device.

The reference models an accelerator in Python (pkg/src/taskbridge/device.py):
in-order queues, completion events, op closures run under a device lock.
Here the same duck type sits on libtb (include/tb.h):

=====================  ===============================  =========================
reference              this module                      libtb
=====================  ===============================  =========================
VirtualDevice          CudaDevice                       tb_init, streams, htq
DeviceQueue.submit     DeviceQueue.submit               async copy/launch + record
DeviceEvent            DeviceEvent (pooled cudaEvent)   tb_event_record/query/wait
DeviceBuffer           DeviceBuffer (HBM + pinned)      tb_malloc / tb_host_alloc
op compute closures    DeviceKernel descriptors         tb_launch / tb_agg_launch
event_wait             CudaDevice.event_wait (fence)    tb_event_wait
register_host_task     CudaDevice.register_host_task    tb_host_task + htq threads
=====================  ===============================  =========================

Only the REAL clock exists (time is the GPU's own). There is no CPU fallback:
constructing a CudaDevice without libtb or a GPU raises.
"""

from __future__ import annotations

import ctypes
import enum
import itertools
import threading
from time import perf_counter
from typing import Callable, Dict, Optional

import numpy as np

from . import _native as N
from .errors import DeviceGoneError, ModeError
from .runtime import _context


class ClockMode(enum.Enum):
    REAL = "real"
    VIRTUAL = "virtual"     # accepted for API parity; a CUDA device rejects it


class OpKind(enum.Enum):
    KERNEL = "kernel"
    COPY_H2D = "h2d"
    COPY_D2H = "d2h"
    BARRIER = "barrier"
    DUMMY = "dummy"


class EventStatus(enum.Enum):
    SUBMITTED = 0
    RUNNING = 1
    COMPLETE = 2


# ----------------------------------------------------------- descriptors --
class DeviceKernel:
    """What a registered kernel kind does to a fused staging buffer.

    Replaces the reference's ``transform(view)`` closures
    (src/executors.py:171-172, src/miniapp.py:40-53): a closure cannot run on
    the GPU, a descriptor can. ``op`` is TB_OP_KIND (built-in kind with the
    reference constants), TB_OP_AFFINE (x*c1 + c2, two roundings) or
    TB_OP_NONE.
    """

    __slots__ = ("op", "kind", "c1", "c2", "name")

    def __init__(self, op: int, kind: int = 0, c1: float = 1.0, c2: float = 0.0,
                 name: str = ""):
        self.op, self.kind, self.c1, self.c2, self.name = op, kind, c1, c2, name

    def __repr__(self):
        return f"DeviceKernel({self.name or self.op})"


def kind_kernel(kind: int) -> DeviceKernel:
    if not 0 <= kind < N.TB_KINDS:
        raise ValueError(f"kernel kind {kind} out of range")
    return DeviceKernel(N.TB_OP_KIND, kind, name=f"kind{kind}")


def affine_kernel(c1: float, c2: float) -> DeviceKernel:
    return DeviceKernel(N.TB_OP_AFFINE, 0, float(c1), float(c2), name=f"affine({c1},{c2})")


NOOP_KERNEL = DeviceKernel(N.TB_OP_NONE, name="noop")


class DeviceBuffer:
    """HBM allocation plus a pinned host mirror used as its staging area.

    ``f64()`` returns the pinned mirror as float64 (the reference's
    ``DeviceBuffer.f64`` is its unified host view, src/device.py:143-154):
    callers marshal into it, an H2D moves it to HBM, a D2H lands results back.
    """

    __slots__ = ("id", "size_bytes", "dptr", "hptr", "host", "_device", "__weakref__")

    def __init__(self, device: "CudaDevice", buf_id: int, size_bytes: int):
        self.id = buf_id
        self.size_bytes = size_bytes
        self._device = device
        d = ctypes.c_void_p()
        N.call("tb_malloc", ctypes.byref(d), size_bytes)
        h = ctypes.c_void_p()
        try:
            N.call("tb_host_alloc", ctypes.byref(h), size_bytes)
        except Exception:
            N.call("tb_free", d)
            raise
        self.dptr, self.hptr = d.value, h.value
        raw = (ctypes.c_uint8 * size_bytes).from_address(self.hptr)
        self.host = np.frombuffer(raw, dtype=np.uint8)

    def f64(self) -> np.ndarray:
        return self.host.view(np.float64)

    def free(self) -> None:
        if self.dptr:
            N.call("tb_free", ctypes.c_void_p(self.dptr))
            N.call("tb_host_free", ctypes.c_void_p(self.hptr))
            self.dptr = self.hptr = 0
            self.host = None


class DeviceEvent:
    """Completion token backed by a pooled cudaEvent (cudaEventDisableTiming).

    Monotone and non-blocking to query, like the reference's DeviceEvent
    (src/device.py:84-103). ``native_handle`` lets the poll registry query it
    in native code. ``completion_time`` is the host time the completion was
    first observed (the device does not timestamp it).
    """

    __slots__ = ("id", "native_handle", "chain", "seq", "completion_time", "_done",
                 "__weakref__")

    _ids = itertools.count()

    def __init__(self, handle: int, chain: int = 0, seq: int = 0):
        self.id = next(DeviceEvent._ids)
        self.native_handle = handle
        self.chain = chain          # the in-order stream it was recorded on
        self.seq = seq              # record order on that stream (1, 2, ...)
        self.completion_time: Optional[float] = None
        self._done = False

    def is_complete(self) -> bool:
        if self._done:
            return True
        if not self.native_handle:
            return False            # parked by a lazy device, not issued yet
        rc = N.fast().tb_event_query(self.native_handle)
        if rc == N.TB_NOT_READY:
            return False
        if rc < 0:
            raise N.CudaError(rc, "tb_event_query")
        self._done = True
        self.completion_time = perf_counter()
        return True

    @property
    def status(self) -> EventStatus:
        return EventStatus.COMPLETE if self.is_complete() else EventStatus.SUBMITTED

    def __del__(self):
        h = self.native_handle
        if h:
            self.native_handle = 0
            try:
                N.fast().tb_event_release(h)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass


class DeviceOp:
    """One queued operation. ``kernel``/``buf``/``host`` describe the payload
    (a closure in the reference, src/device.py:106-121)."""

    __slots__ = ("kind", "work_items", "nbytes", "kernel", "buf", "host", "spin_ns",
                 "event", "queue", "index")

    def __init__(self, kind: OpKind, work_items: int = 0, nbytes: int = 0,
                 kernel: Optional[DeviceKernel] = None, buf=None, host=None,
                 spin_ns: int = 0):
        self.kind = kind
        self.work_items = work_items
        self.nbytes = nbytes
        self.kernel = kernel
        self.buf = buf
        self.host = host
        self.spin_ns = spin_ns
        self.event: Optional[DeviceEvent] = None
        self.queue = None
        self.index: Optional[int] = None


def make_kernel(work_items: int, kernel: Optional[DeviceKernel] = None,
                buf: Optional[DeviceBuffer] = None) -> DeviceOp:
    """A kernel over ``work_items`` doubles of ``buf`` (no buffer: empty kernel)."""
    return DeviceOp(OpKind.KERNEL, work_items=work_items, kernel=kernel, buf=buf)


def make_spin(microseconds: float) -> DeviceOp:
    """A kernel that keeps its queue busy for the given time (device-side
    %globaltimer spin); stands in for the reference tests' long gate ops."""
    return DeviceOp(OpKind.KERNEL, spin_ns=int(microseconds * 1e3))


def make_h2d(nbytes: int, dst: Optional[DeviceBuffer] = None, src=None) -> DeviceOp:
    """Copy ``nbytes`` from host ``src`` (default: dst's pinned mirror) to HBM."""
    return DeviceOp(OpKind.COPY_H2D, nbytes=nbytes, buf=dst, host=src)


def make_d2h(nbytes: int, src: Optional[DeviceBuffer] = None, dst=None) -> DeviceOp:
    """Copy ``nbytes`` from HBM to host ``dst`` (default: src's pinned mirror)."""
    return DeviceOp(OpKind.COPY_D2H, nbytes=nbytes, buf=src, host=dst)


def make_barrier() -> DeviceOp:
    return DeviceOp(OpKind.BARRIER)


def make_dummy() -> DeviceOp:
    return DeviceOp(OpKind.DUMMY)


def _host_ptr(host, buf: Optional[DeviceBuffer]) -> int:
    if host is None:
        return buf.hptr
    if isinstance(host, np.ndarray):
        if not host.flags.c_contiguous:
            raise ValueError("host array must be C-contiguous")
        return host.ctypes.data
    return int(host)


class DeviceQueue:
    """In-order queue = one non-blocking CUDA stream (src/device.py:157-180)."""

    __slots__ = ("device", "id", "stream", "_submit_count", "_record_count", "_lock")

    def __init__(self, device: "CudaDevice", queue_id: int):
        self.device = device
        self.id = queue_id
        h = ctypes.c_uint64(0)
        N.call("tb_stream_create", ctypes.byref(h))
        self.stream = h.value
        self._submit_count = 0
        self._record_count = 0      # events recorded, under _lock (poll-chain order)
        self._lock = threading.Lock()

    @property
    def in_order(self) -> bool:
        return True

    def submit(self, op: DeviceOp) -> DeviceEvent:
        return self.device._submit(self, op)

    def incomplete_count(self) -> int:
        return 1 if N.fast().tb_stream_query(self.stream) == N.TB_NOT_READY else 0


class _Counters:
    __slots__ = ("kernels", "h2d", "d2h", "barriers", "barriers_elided", "dummies",
                 "event_waits", "hosttask_dispatched")

    def __init__(self):
        for f in self.__slots__:
            setattr(self, f, 0)

    def snapshot(self) -> dict:
        d = {f: getattr(self, f) for f in self.__slots__}
        d["transfers"] = d["h2d"] + d["d2h"]
        return d


class CudaDevice:
    """One GPU as seen by the task runtime (duck type of VirtualDevice,
    src/device.py:196-401).

    ``compute_slots`` is accepted for API parity; kernel concurrency is the
    hardware's. ``barrier_elision`` skips BARRIER launches (their event rides
    on the queue tail, src/device.py:419-432); ``event_pool`` toggles libtb's
    event pool (src/device.py:221,410-411). Host tasks are dispatched by
    ``hosttask_threads`` Python threads named ``tb-hosttask-i`` fed by libtb's
    host-task queue (stream callbacks on side streams). ``record_timeline``
    brackets every op with CUDA timing events and exposes the reference's
    (queue, index, kind, start, completion) rows as ``timeline``.
    ``latency`` and ``hosttask_dispatch_cost`` belong to the reference's
    simulator (the hardware has its own) and are ignored; the virtual clock
    lives in the CPU test double (tests/virtual_device.py).
    """

    def __init__(self, device_index: int = 0, compute_slots: int = 16,
                 clock_mode: ClockMode = ClockMode.REAL, latency=None,
                 hosttask_threads: int = 2, hosttask_dispatch_cost: float = 0.0,
                 barrier_elision: bool = False, lazy_submit: bool = False,
                 event_pool: bool = True, record_timeline: bool = False,
                 hosttask_side_streams: int = 4):
        if clock_mode is not ClockMode.REAL:
            raise ModeError("a CUDA device runs on the real clock only")
        if compute_slots < 1:
            raise ValueError("compute_slots must be >= 1")
        N.init(device_index)
        N.call("tb_event_pool_set", 1 if event_pool else 0)
        self.device_index = device_index
        self.compute_slots = compute_slots
        self.clock_mode = clock_mode
        self.latency = latency
        self.barrier_elision = barrier_elision
        # Lazy submit (src/device.py:441-453, the hipSYCL flush workaround,
        # PAPER.md:587-600): ops park on the host until flush() — which the
        # Integration installs as a poll-registry flush hook — issues them.
        self.lazy_submit = lazy_submit
        self._held: list = []            # (queue, op, placeholder event, issue fn)
        self.event_pool = event_pool
        self.record_timeline = record_timeline
        self._timeline_rows: list = []      # resolved (queue, index, kind, start, completion)
        self._timeline_pending: list = []   # (queue id, index, kind, start ev, end ev)
        self._epoch = 0
        self.counters = _Counters()
        self._lock = threading.Lock()
        self._alive = True
        self._queues: list = []
        self._buffer_ids = itertools.count()
        self._buffers: list = []
        if record_timeline:
            # the timeline's t = 0: a timing event on a private stream; op
            # times are elapsed times from it (seconds, like the reference's
            # virtual clock, src/device.py:223-224,512-514)
            h = ctypes.c_uint64(0)
            N.call("tb_stream_create", ctypes.byref(h))
            self._epoch_stream = h.value
            e = ctypes.c_uint64(0)
            N.call("tb_tevent_record", self._epoch_stream, ctypes.byref(e))
            N.call("tb_stream_sync", self._epoch_stream)
            self._epoch = e.value
        # host tasks
        h = ctypes.c_uint64(0)
        N.call("tb_htq_create", hosttask_side_streams, ctypes.byref(h))
        self._htq = h.value
        self._ht_lock = threading.Lock()
        self._ht_entries: Dict[int, tuple] = {}
        self._ht_tokens = itertools.count(1)
        self._ht_active = 0
        self._ht_threads = [threading.Thread(target=self._hosttask_loop,
                                             name=f"tb-hosttask-{i}", daemon=True)
                            for i in range(hosttask_threads)]
        for t in self._ht_threads:
            t.start()

    # ------------------------------------------------------------- public --
    def queue(self) -> DeviceQueue:
        with self._lock:
            if not self._alive:
                raise DeviceGoneError("device destroyed")
            q = DeviceQueue(self, len(self._queues))
            self._queues.append(q)
            return q

    def alloc_buffer(self, size_bytes: int) -> DeviceBuffer:
        if size_bytes <= 0:
            raise ValueError("size_bytes must be > 0")
        buf = DeviceBuffer(self, next(self._buffer_ids), size_bytes)
        with self._lock:
            self._buffers.append(buf)
        return buf

    def now(self) -> float:
        return perf_counter()

    def set_barrier_elision(self, enabled: bool) -> None:
        self.barrier_elision = enabled

    def event_status(self, event: DeviceEvent) -> EventStatus:
        if self.lazy_submit and not event.native_handle:
            self.flush()            # first status query kicks the lazy scheduler
        return event.status

    def event_wait(self, event: DeviceEvent) -> None:
        """Block the calling thread until ``event`` completes (FENCE)."""
        with self._lock:
            self.counters.event_waits += 1
            if not self._alive:
                raise DeviceGoneError("device destroyed while waiting")
        if self.lazy_submit and not event.native_handle:
            self.flush()
        if event.is_complete():
            return
        worker = _context.current_worker()
        pool = worker.pool if worker is not None else None
        if pool is not None:
            pool._note_blocked(+1)
        try:
            rc = N.blocking().tb_event_wait(event.native_handle)
        finally:
            if pool is not None:
                pool._note_blocked(-1)
        if rc < 0:
            raise N.CudaError(rc, "tb_event_wait")
        if not self._alive:
            raise DeviceGoneError("device destroyed while waiting")
        event.is_complete()

    def register_host_task(self, event: DeviceEvent, cb: Callable[[], None],
                           on_abandon: Optional[Callable] = None) -> None:
        if self.lazy_submit and not event.native_handle:
            self.flush()
        with self._ht_lock:
            if not self._alive:
                raise DeviceGoneError("device destroyed")
            token = next(self._ht_tokens)
            self._ht_entries[token] = (cb, on_abandon)
        rc = N.fast().tb_host_task(self._htq, event.native_handle, token)
        if rc < 0:
            with self._ht_lock:
                self._ht_entries.pop(token, None)
            if rc == N.TB_E_CLOSED:
                raise DeviceGoneError("device destroyed")
            raise N.CudaError(rc, "tb_host_task")

    def flush(self) -> None:
        """Issue every op parked by lazy submit, in submission order."""
        if not self.lazy_submit:
            return
        with self._lock:
            held, self._held = self._held, []
        for queue, op, ev, issue in held:
            real = issue()
            # hand the recorded CUDA event to the placeholder callers hold
            ev.native_handle, real.native_handle = real.native_handle, 0
            ev.chain, ev.seq = real.chain, real.seq
            if op is not None:
                op.event = ev

    def has_pending(self) -> bool:
        """Ops issued to the GPU and not yet complete (parked ops excluded,
        as in the reference's lazy mode, src/device.py:355-357)."""
        return any(q.incomplete_count() for q in self._queues)

    def held_count(self) -> int:
        with self._lock:
            return len(self._held)

    def hosttask_backlog(self) -> int:
        with self._ht_lock:
            return len(self._ht_entries)

    def hosttask_thread_set(self) -> set:
        return set(self._ht_threads)

    def snapshot_counters(self) -> dict:
        with self._lock:
            return self.counters.snapshot()

    def synchronize(self) -> None:
        N.call("tb_device_sync")

    def destroy(self) -> None:
        with self._lock:
            if not self._alive:
                return
            self._alive = False
        with self._ht_lock:
            abandoned = list(self._ht_entries.values())
            self._ht_entries.clear()
        N.call("tb_htq_close", self._htq)
        for _cb, on_abandon in abandoned:
            if on_abandon is not None:
                try:
                    on_abandon(DeviceGoneError("device destroyed"))
                except BaseException:  # noqa: BLE001
                    pass
        for t in self._ht_threads:
            if t is not threading.current_thread():
                t.join(timeout=2.0)
        N.call("tb_htq_destroy", self._htq)
        try:
            N.call("tb_device_sync")
            if self.record_timeline:
                for *_, a, b in self._timeline_pending:
                    N.fast().tb_tevent_release(a)
                    N.fast().tb_tevent_release(b)
                self._timeline_pending = []
                N.fast().tb_tevent_release(self._epoch)
                N.call("tb_stream_destroy", self._epoch_stream)
        finally:
            for q in self._queues:
                N.call("tb_stream_destroy", q.stream)
            for b in self._buffers:
                b.free()
            self._buffers.clear()

    # ---------------------------------------------------------- timeline --
    @property
    def timeline(self) -> list:
        """(queue, index, kind, start, completion) per completed op, seconds
        from the device's creation, in completion order — the reference's
        record_timeline rows (src/device.py:512-514), from CUDA timing events
        recorded around every op."""
        if not self.record_timeline:
            return []
        with self._lock:
            pending, self._timeline_pending = self._timeline_pending, []
            keep = []
            ms0, ms1 = ctypes.c_double(0.0), ctypes.c_double(0.0)
            for row in pending:
                qid, idx, kind, a, b = row
                r0 = N.fast().tb_tevent_elapsed(self._epoch, a, ctypes.byref(ms0))
                r1 = N.fast().tb_tevent_elapsed(self._epoch, b, ctypes.byref(ms1))
                if r0 == N.TB_NOT_READY or r1 == N.TB_NOT_READY:
                    keep.append(row)
                    continue
                if r0 < 0 or r1 < 0:
                    raise N.CudaError(min(r0, r1), "tb_tevent_elapsed")
                self._timeline_rows.append((qid, idx, kind, ms0.value * 1e-3, ms1.value * 1e-3))
                N.fast().tb_tevent_release(a)
                N.fast().tb_tevent_release(b)
            self._timeline_pending = keep + self._timeline_pending
            self._timeline_rows.sort(key=lambda r: (r[4], r[0], r[1]))
            return list(self._timeline_rows)

    def _mark(self, queue: DeviceQueue) -> int:
        """A timing event on ``queue`` now (record_timeline only)."""
        e = ctypes.c_uint64(0)
        rc = N.fast().tb_tevent_record(queue.stream, ctypes.byref(e))
        if rc < 0:
            raise N.CudaError(rc, "tb_tevent_record")
        return e.value

    # ------------------------------------------------------------ engine --
    def _record(self, queue: DeviceQueue) -> DeviceEvent:
        """Record an event on ``queue`` (caller holds ``queue._lock``): its
        sequence number orders it in the poll registry's chain for the
        stream, whatever order producers register in."""
        h = ctypes.c_uint64(0)
        rc = N.fast().tb_event_record(queue.stream, ctypes.byref(h))
        if rc < 0:
            raise N.CudaError(rc, "tb_event_record")
        queue._record_count += 1
        return DeviceEvent(h.value, queue.stream, queue._record_count)

    def _park(self, queue: DeviceQueue, op, issue) -> DeviceEvent:
        ev = DeviceEvent(0)
        if op is not None:
            op.event = ev
        with self._lock:
            self._held.append((queue, op, ev, issue))
        return ev

    def _submit(self, queue: DeviceQueue, op: DeviceOp) -> DeviceEvent:
        if op.queue is not None:
            raise ValueError("op already submitted")
        if not self._alive:
            raise DeviceGoneError("device destroyed")
        if self.lazy_submit:
            op.queue = queue
            return self._park(queue, op, lambda: self._issue(queue, op))
        return self._issue(queue, op)

    def _issue(self, queue: DeviceQueue, op: DeviceOp) -> DeviceEvent:
        c = self.counters
        s = queue.stream
        with queue._lock:
            op.queue = queue
            op.index = queue._submit_count
            queue._submit_count += 1
            k = op.kind
            t0 = self._mark(queue) if self.record_timeline else 0
            if k is OpKind.KERNEL:
                if op.spin_ns:
                    N.call("tb_spin", s, op.spin_ns)
                elif op.buf is not None and op.kernel is not None:
                    kd = op.kernel
                    N.call("tb_launch", s, kd.op, kd.kind, kd.c1, kd.c2,
                           op.buf.dptr, op.work_items)
                else:
                    N.call("tb_launch", s, N.TB_OP_NONE, 0, 1.0, 0.0, None, 0)
                with self._lock:
                    c.kernels += 1
            elif k is OpKind.COPY_H2D:
                N.call("tb_memcpy_h2d", s, op.buf.dptr, _host_ptr(op.host, op.buf),
                       op.nbytes)
                with self._lock:
                    c.h2d += 1
            elif k is OpKind.COPY_D2H:
                N.call("tb_memcpy_d2h", s, _host_ptr(op.host, op.buf), op.buf.dptr,
                       op.nbytes)
                with self._lock:
                    c.d2h += 1
            elif k is OpKind.BARRIER:
                if self.barrier_elision:
                    with self._lock:
                        c.barriers_elided += 1
                else:
                    N.call("tb_barrier", s)
                    with self._lock:
                        c.barriers += 1
            else:
                with self._lock:
                    c.dummies += 1
            if self.record_timeline and not (k is OpKind.BARRIER and self.barrier_elision):
                t1 = self._mark(queue)
                with self._lock:
                    self._timeline_pending.append((queue.id, op.index, k.value, t0, t1))
            elif t0:
                N.fast().tb_tevent_release(t0)
            op.event = self._record(queue)
        return op.event

    def submit_batch(self, queue: DeviceQueue, kernel: DeviceKernel,
                     staging: DeviceBuffer, nbytes: int, barrier: bool) -> DeviceEvent:
        """One aggregated launch (src/executors.py:257-284) in one native call:
        H2D(staging) ; kernel ; [barrier] ; D2H(staging) ; record."""
        if not self._alive:
            raise DeviceGoneError("device destroyed")
        if self.lazy_submit:
            return self._park(queue, None, lambda: self._issue_batch(
                queue, kernel, staging, nbytes, barrier))
        return self._issue_batch(queue, kernel, staging, nbytes, barrier)

    def _issue_batch_timed(self, queue: DeviceQueue, kernel: DeviceKernel,
                           staging: DeviceBuffer, nbytes: int, barrier: bool,
                           do_barrier: bool) -> int:
        """The batch's ops one call each, timing events around each op
        (record_timeline): one timeline row per op as in the reference
        (H2D, KERNEL, [BARRIER], D2H: src/executors.py:277-284)."""
        s = queue.stream
        ops = [("h2d", lambda: N.call("tb_memcpy_h2d", s, staging.dptr, staging.hptr, nbytes)),
               ("kernel", lambda: N.call("tb_launch", s, kernel.op, kernel.kind, kernel.c1,
                                         kernel.c2, staging.dptr, nbytes // 8))]
        if barrier and do_barrier:
            ops.append(("barrier", lambda: N.call("tb_barrier", s)))
        ops.append(("d2h", lambda: N.call("tb_memcpy_d2h", s, staging.hptr, staging.dptr,
                                          nbytes)))
        rows = []
        index = queue._submit_count
        for kind, issue in ops:
            if kind == "d2h" and barrier and not do_barrier:
                index += 1                      # the elided barrier's index
            start = self._mark(queue)           # each row owns its two events
            issue()
            rows.append((queue.id, index, kind, start, self._mark(queue)))
            index += 1
        with self._lock:
            self._timeline_pending.extend(rows)
        h = ctypes.c_uint64(0)
        rc = N.fast().tb_event_record(s, ctypes.byref(h))
        if rc < 0:
            raise N.CudaError(rc, "tb_event_record")
        return h.value

    def _issue_batch(self, queue: DeviceQueue, kernel: DeviceKernel,
                     staging: DeviceBuffer, nbytes: int, barrier: bool) -> DeviceEvent:
        do_barrier = barrier and not self.barrier_elision
        h = ctypes.c_uint64(0)
        if self.record_timeline:
            with queue._lock:
                h.value = self._issue_batch_timed(queue, kernel, staging, nbytes, barrier,
                                                  do_barrier)
                queue._submit_count += 4 if barrier else 3
                queue._record_count += 1
                seq = queue._record_count
            return self._count_batch(DeviceEvent(h.value, queue.stream, seq), barrier,
                                     do_barrier)
        with queue._lock:
            rc = N.fast().tb_agg_launch(queue.stream, kernel.op, kernel.kind,
                                            kernel.c1, kernel.c2, staging.dptr,
                                            staging.hptr, nbytes,
                                            1 if do_barrier else 0, ctypes.byref(h))
            queue._submit_count += 4 if barrier else 3
            if rc >= 0:
                queue._record_count += 1
                seq = queue._record_count
        if rc < 0:
            raise N.CudaError(rc, "tb_agg_launch")
        return self._count_batch(DeviceEvent(h.value, queue.stream, seq), barrier, do_barrier)

    def _count_batch(self, ev: DeviceEvent, barrier: bool, do_barrier: bool) -> DeviceEvent:
        with self._lock:
            c = self.counters
            c.h2d += 1
            c.kernels += 1
            c.d2h += 1
            if barrier:
                if do_barrier:
                    c.barriers += 1
                else:
                    c.barriers_elided += 1
        return ev

    # -------------------------------------------------------- host tasks --
    def _hosttask_loop(self) -> None:
        tok = ctypes.c_uint64(0)
        status = ctypes.c_int(0)
        lib = N.blocking()
        while True:
            rc = lib.tb_htq_next(self._htq, ctypes.byref(tok), ctypes.byref(status), 50_000)
            if rc == N.TB_E_CLOSED:
                return
            if rc != N.TB_OK:
                if not self._alive:
                    return
                continue
            with self._ht_lock:
                entry = self._ht_entries.pop(tok.value, None)
                if entry is not None:
                    self._ht_active += 1
            if entry is None:
                continue
            try:
                if status.value < 0:
                    # the device faulted before the event: fault the future
                    # (src/executors.py:50-55), never run the completion
                    if entry[1] is not None:
                        entry[1](N.CudaError(status.value, "device fault before host task"))
                else:
                    entry[0]()
            except BaseException:  # noqa: BLE001 - callback faults land in futures
                pass
            finally:
                with self._ht_lock:
                    self._ht_active -= 1
                with self._lock:
                    self.counters.hosttask_dispatched += 1


# The reference name, for callers that construct "the device" generically.
VirtualDevice = CudaDevice
