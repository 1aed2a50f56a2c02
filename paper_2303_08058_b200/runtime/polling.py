"""Event-callback registry polled by the scheduler between tasks.

Same contract as the reference registry (pkg/src/taskbridge/runtime/polling.py):
producers ``add`` from any thread without taking a lock; ``poll`` is
single-entrant — a contender fails the guard and returns 0 at once — drains
new registrations, re-checks pending ones and fires callbacks whose event is
complete; ``abandon_all`` fails every unfired entry at shutdown (fired
callbacks for already-complete events still run).

B200 design: entries whose event carries a CUDA handle (``native_handle``)
go straight into libtb's native registry (tb_poll_add: lock-free MPSC
push, keyed by the event's in-order stream); ``poll`` then checks them with
one non-blocking native call — only the head of each stream's FIFO is
queried — that returns the fired tokens, with the GIL held throughout.
Events without a native handle (e.g. test doubles exposing only
``is_complete()``, the only contract the reference relies on —
pkg/tests/conftest.py:35-44) use a Python-side inbox/pending list.
"""

from __future__ import annotations

import ctypes
import itertools
import threading
from collections import deque
from typing import Callable, Dict, Optional

from .. import _native as N


class EventCallback:
    """An event paired with what to run once it completes (or on abandon)."""

    __slots__ = ("event", "callback", "on_abandon")

    def __init__(self, event, callback: Callable[[], None], on_abandon=None):
        self.event = event
        self.callback = callback
        self.on_abandon: Optional[Callable[[BaseException], None]] = on_abandon


_FIRE_CAP = 4096


class PollRegistry:
    def __init__(self):
        self._inbox: deque = deque()           # python-path entries
        self._pending: list = []
        self._guard = threading.Lock()
        self._entry_lock = threading.Lock()
        self._entries = 0
        self.entry_high_water = 0
        self.fired_total = 0
        self._flush_hooks: list = []
        self._enter: Optional[Callable[[], None]] = None
        self._exit: Optional[Callable[[], None]] = None
        # native path
        self._native = None                      # tb_poll_t, created lazily
        self._native_lock = threading.Lock()
        self._tokens: Dict[int, EventCallback] = {}
        self._next_token = itertools.count(1)
        self._fired_buf = None
        self._status_buf = None

    # ------------------------------------------------------------- config --
    def set_activity_hooks(self, enter, exit) -> None:
        self._enter, self._exit = enter, exit

    def add_flush_hook(self, fn: Callable[[], None]) -> None:
        self._flush_hooks.append(fn)

    # ---------------------------------------------------------- producers --
    def _native_reg(self):
        if self._native is None:
            with self._native_lock:
                if self._native is None:
                    h = ctypes.c_uint64(0)
                    N.call("tb_poll_create", ctypes.byref(h))
                    self._fired_buf = (ctypes.c_uint64 * _FIRE_CAP)()
                    self._status_buf = (ctypes.c_int32 * _FIRE_CAP)()
                    self._native = h.value
        return self._native

    def add(self, ec: EventCallback) -> None:
        handle = getattr(ec.event, "native_handle", None)
        if handle:
            reg = self._native_reg()
            token = next(self._next_token)
            self._tokens[token] = ec
            rc = N.fast().tb_poll_add_seq(reg, handle, getattr(ec.event, "chain", 0),
                                          getattr(ec.event, "seq", 0), token)
            if rc != 0:
                del self._tokens[token]
                raise N.CudaError(rc, "tb_poll_add")
            return
        self._inbox.append(ec)

    # -------------------------------------------------------------- gauges --
    def inbox_size(self) -> int:
        return len(self._inbox)

    def pending_count(self) -> int:
        return len(self._pending) + len(self._tokens)

    def has_waiting(self) -> bool:
        return bool(self._inbox) or bool(self._pending) or bool(self._tokens)

    # ---------------------------------------------------------- poll body --
    def _run(self, ec: EventCallback) -> None:
        enter, leave = self._enter, self._exit
        if enter is not None:
            enter()
        try:
            ec.callback()
        except BaseException:  # noqa: BLE001 - the producer's future carries faults
            pass
        finally:
            if leave is not None:
                leave()

    def poll(self) -> int:
        """Fire callbacks of completed events; 0 at once if another thread polls."""
        if not self._guard.acquire(blocking=False):
            return 0
        with self._entry_lock:
            self._entries += 1
            if self._entries > self.entry_high_water:
                self.entry_high_water = self._entries
        fired = 0
        try:
            for hook in self._flush_hooks:
                hook()
            if self._tokens:
                fired += self._poll_native()
            if self._inbox or self._pending:
                fired += self._poll_python()
            self.fired_total += fired
        finally:
            with self._entry_lock:
                self._entries -= 1
            self._guard.release()
        return fired

    def _fault(self, ec: EventCallback, error: BaseException) -> None:
        """A device fault behind ``ec``'s event: its future faults (the
        callback, which would read the op's garbage outputs, never runs)."""
        if ec.on_abandon is not None:
            try:
                ec.on_abandon(error)
            except BaseException:  # noqa: BLE001
                pass

    def _poll_native(self) -> int:
        n = ctypes.c_int(0)
        buf, status = self._fired_buf, self._status_buf
        # GIL held: the native body never blocks, and releasing the GIL here
        # would let a busy worker keep it for a whole switch interval.
        rc = N.fast().tb_poll(self._native, buf, status, _FIRE_CAP, ctypes.byref(n))
        if rc < 0:
            raise N.CudaError(rc, "tb_poll")
        k = n.value
        pop = self._tokens.pop
        for i in range(k):
            ec = pop(buf[i])
            if status[i] < 0:
                self._fault(ec, N.CudaError(status[i], "device fault before event"))
            else:
                self._run(ec)
        return k

    def _complete(self, ec: EventCallback):
        """True/False = event complete or not; None = the query faulted (the
        entry is then faulted and dropped)."""
        try:
            return ec.event.is_complete()
        except BaseException as e:  # noqa: BLE001 - device fault
            self._fault(ec, e)
            return None

    def _poll_python(self) -> int:
        fired = 0
        still = []
        for ec in self._pending:                 # older registrations first
            done = self._complete(ec)
            if done:
                self._run(ec)
            if done is not False:
                fired += 1
            else:
                still.append(ec)
        while True:
            try:
                ec = self._inbox.popleft()
            except IndexError:
                break
            done = self._complete(ec)
            if done:
                self._run(ec)
            if done is not False:
                fired += 1
            else:
                still.append(ec)
        self._pending = still
        return fired

    # ------------------------------------------------------------ shutdown --
    def abandon_all(self, error: BaseException) -> int:
        abandoned = 0
        with self._guard:
            entries = [(ec, self._complete(ec)) for ec in self._pending]
            self._pending = []
            while self._inbox:
                ec = self._inbox.popleft()
                entries.append((ec, self._complete(ec)))
            if self._native is not None:
                cap = max(1, len(self._tokens))
                toks = (ctypes.c_uint64 * cap)()
                done = (ctypes.c_uint8 * cap)()
                n = ctypes.c_int(0)
                N.call("tb_poll_drain", self._native, toks, done, cap, ctypes.byref(n))
                for i in range(n.value):
                    ec = self._tokens.pop(toks[i])
                    if done[i] == 2:        # the device faulted before it
                        self._fault(ec, N.CudaError(-1, "device fault before event"))
                        entries.append((ec, None))
                    else:
                        entries.append((ec, bool(done[i])))
            for ec, complete in entries:
                if complete is None:            # faulted above
                    continue
                if complete:
                    self._run(ec)
                    continue
                abandoned += 1
                if ec.on_abandon is not None:
                    try:
                        ec.on_abandon(error)
                    except BaseException:  # noqa: BLE001
                        pass
        return abandoned

    def close(self) -> None:
        if self._native is not None:
            N.call("tb_poll_destroy", self._native)
            self._native = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
