"""Independent timeline oracle for the virtual-clock double — TEST
INFRASTRUCTURE (criterion 9, pkg/tests/test_acceptance.py:204-241).

Given a script of ops all submitted at t = 0 in script order, computes the
(queue, index, kind, start, completion) row of every op under the documented
queue semantics, with none of the engine's data structures (no heaps, no
queue objects, no parked list): a calendar of pending completions kept as a
sorted Python list, and a "who may start" rule re-evaluated after every
completion:

* a queue's next op may start once its previous op has completed;
* copies, barriers and markers start at once; a kernel needs one of the
  ``slots`` compute slots;
* after a completion, the queue that completed goes first (it may take the
  slot just freed), then kernels that had to wait, oldest wait first, ties
  by queue id;
* completions at the same instant are handled in the order their ops
  started.
"""

from __future__ import annotations

import bisect
from typing import Dict, List, Tuple

Row = Tuple[int, int, str, float, float]


def op_time(kind: str, items: int, nbytes: int, lat) -> float:
    return {"kernel": lat.kernel_fixed + lat.kernel_per_item * items,
            "h2d": lat.copy_per_byte * nbytes,
            "d2h": lat.copy_per_byte * nbytes,
            "barrier": lat.barrier_cost}.get(kind, lat.kernel_fixed)


def timeline(script, lat, slots: int) -> List[Row]:
    todo: Dict[int, List[Tuple[int, str, int, int]]] = {}
    for q, kind, items, nbytes in script:
        todo.setdefault(q, []).append((len(todo.get(q, [])), kind, items, nbytes))
    cursor = {q: 0 for q in todo}          # next op index per queue
    busy = set()                           # queues with an op in flight
    calendar: List[tuple] = []             # sorted (end, started_as, q, idx, kind, start)
    waiting_since: Dict[int, float] = {}   # queue -> time its kernel began waiting
    used = 0
    started = 0
    rows: List[Row] = []

    def ready(q):
        return q not in busy and cursor[q] < len(todo[q])

    def launch(q, t):
        nonlocal used, started
        idx, kind, items, nbytes = todo[q][cursor[q]]
        cursor[q] += 1
        busy.add(q)
        if kind == "kernel":
            used += 1
        bisect.insort(calendar, (t + op_time(kind, items, nbytes, lat), started, q, idx, kind, t))
        started += 1

    def offer(q, t):
        """Start q's next op if it may; a blocked kernel starts waiting."""
        if not ready(q):
            return
        if todo[q][cursor[q]][1] == "kernel" and used >= slots:
            waiting_since.setdefault(q, t)
            return
        waiting_since.pop(q, None)
        launch(q, t)

    for q, *_ in script:                   # every submit offers its queue
        offer(q, 0.0)
    while calendar:
        end, _, q, idx, kind, start = calendar.pop(0)
        rows.append((q, idx, kind, start, end))
        busy.discard(q)
        if kind == "kernel":
            used -= 1
        offer(q, end)
        for w in sorted(waiting_since, key=lambda k: (waiting_since[k], k)):
            if used >= slots:
                break
            if ready(w):
                del waiting_since[w]
                launch(w, end)
    return rows
