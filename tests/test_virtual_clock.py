"""Acceptance criteria 8 and 9 of the reference kept
testable on CPU with the virtual-clock device double (tests/virtual_device.py)
and an independent timeline oracle (tests/timeline_oracle.py):

* criterion 8 — two identical virtual-clock sweeps through the benchmark CLI
  write byte-identical CSVs (pkg/tests/test_acceptance.py:190-202);
* criterion 9 — a two-queue, one-slot script produces the same
  (queue, index, kind, start, completion) timeline as the independent oracle
  (pkg/tests/test_acceptance.py:204-241).

Plus the machine on the virtual clock: the reference goldens in every
completion mode, the unfused counts, and the modelled step times (the
reference's virtual-mode numbers: SURVEY.md §6, polling 15.36 ms with 960
launches at 512 sub-grids)."""

import itertools
import random

import pytest

from conftest import fx
from paper_2303_08058_b200 import (AggregationExecutor, BufferPool, ExecutorPool,
                                   Integration, IntegrationMode, Runtime, ScenarioConfig,
                                   build_scenario, cli, kernel_transform, run_scenario)
from paper_2303_08058_b200.device import (make_barrier, make_d2h, make_dummy, make_h2d,
                                          make_kernel)
from timeline_oracle import timeline
from virtual_device import Latency, VirtualClockDevice, VirtualClockPump, make_virtual_stack

MODES = list(IntegrationMode)


def test_criterion_8_virtual_sweeps_are_byte_identical(tmp_path):
    argv = ["--clock", "virtual", "--subgrids", "4", "--steps", "2",
            "--executors", "2", "--max-agg", "4", "--sweep", "workers"]
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    assert cli.main(argv + ["--out", str(a)], devices=make_virtual_stack()) == cli.EXIT_OK
    assert cli.main(argv + ["--out", str(b)], devices=make_virtual_stack()) == cli.EXIT_OK
    ta, tb = a.read_bytes(), b.read_bytes()
    assert ta == tb
    rows = ta.decode().splitlines()
    assert len(rows) == 1 + 4          # header + one row per worker count
    # every row carries the reference checksum of run_reference(4, 2)
    assert {r.split(",")[-1] for r in rows[1:]} == {"0x1.8e6968eb86d56p+10"}


SCRIPT = [(0, "kernel", 512, 0), (1, "kernel", 300, 0), (0, "h2d", 8192, 0),
          (1, "kernel", 100, 0), (0, "kernel", 1024, 0), (1, "d2h", 2048, 0),
          (0, "barrier", 0, 0), (1, "barrier", 0, 0), (0, "d2h", 8192, 0),
          (1, "kernel", 700, 0)]
MAKERS = {"kernel": lambda it, nb: make_kernel(it), "h2d": lambda it, nb: make_h2d(nb),
          "d2h": lambda it, nb: make_d2h(nb), "barrier": lambda it, nb: make_barrier(),
          "dummy": lambda it, nb: make_dummy()}


def run_script(script, slots, nq):
    lat = Latency()
    dev = VirtualClockDevice(compute_slots=slots, latency=lat, record_timeline=True)
    try:
        qs = [dev.queue() for _ in range(nq)]
        for q, kind, items, nbytes in script:
            qs[q].submit(MAKERS[kind](items, nbytes))
        while dev.advance_to_next():
            pass
        return dev.timeline, lat
    finally:
        dev.destroy()


def test_criterion_9_two_queue_timeline_matches_oracle():
    got, lat = run_script(SCRIPT, 1, 2)
    assert len(got) == len(SCRIPT)
    assert got == timeline(SCRIPT, lat, 1)


@pytest.mark.parametrize("seed", range(12))
def test_random_timelines_match_oracle(seed):
    rng = random.Random(seed)
    nq = rng.randint(1, 5)
    slots = rng.randint(1, 3)
    kinds = ["kernel", "kernel", "h2d", "d2h", "barrier", "dummy"]
    script = [(rng.randrange(nq), k, rng.choice([0, 64, 512, 4096]), rng.choice([0, 4096]))
              for k in (rng.choice(kinds) for _ in range(rng.randint(5, 40)))]
    got, lat = run_script(script, slots, nq)
    assert got == timeline(script, lat, slots)


class VStack:
    def __init__(self, workers=2, executors=2, max_agg=8, mode=IntegrationMode.POLLING,
                 slots=16, barrier_elision=False):
        self.runtime = Runtime(workers, seed=11)
        self.device = VirtualClockDevice(compute_slots=slots, barrier_elision=barrier_elision)
        integ = Integration(self.runtime, self.device, mode)
        pool = ExecutorPool(integ, executors)
        bufs = BufferPool(self.device)
        self.aggs = [AggregationExecutor(ex, max_agg, bufs) for ex in pool.executors]
        for a in self.aggs:
            for k in range(5):
                a.register_kind(k, kernel_transform(k))

    def run(self, subgrids, steps):
        sc = build_scenario(ScenarioConfig(subgrids=subgrids, steps=steps))
        by_grid = [self.aggs[g % len(self.aggs)] for g in range(subgrids)]
        pump = VirtualClockPump(self.runtime, self.device, 60.0)
        return run_scenario(sc, self.runtime, self.device, self.aggs, by_grid, pump=pump)

    def close(self):
        self.runtime.shutdown()
        self.device.destroy()


@pytest.fixture
def vstack():
    made = []

    def make(**kw):
        s = VStack(**kw)
        made.append(s)
        return s

    yield make
    for s in made:
        s.close()


@pytest.mark.parametrize("mode", MODES)
def test_virtual_machine_goldens_every_mode(vstack, golden, mode):
    lit = golden["reference_test_literals"]
    res = vstack(mode=mode).run(4, 2)
    assert res.checksum == fx(lit["GOLDEN_4X2"])
    assert res.dts == [fx(h) for h in lit["GOLDEN_4X2_DTS"]]
    # virtual step times are device time: positive, and repeatable
    again = vstack(mode=mode).run(4, 2)
    assert [m.wall_ms for m in res.per_step] == [m.wall_ms for m in again.per_step]
    assert all(m.wall_ms > 0 for m in res.per_step)


def test_virtual_unfused_counts_and_fence_batches(vstack, golden):
    res = vstack(executors=1, max_agg=1).run(8, 2)
    for m in res.per_step:
        assert m.launches == 8 * 15 and m.transfers == 8 * 30
    assert res.checksum == fx(golden["reference_test_literals"]["GOLDEN_8X2"])
    # fence: the idleness probe blocks the scheduling worker until the queue
    # drains, so every batch launches alone
    f = vstack(executors=2, max_agg=8, mode=IntegrationMode.FENCE).run(8, 1)
    assert all(sz == 1 for m in f.per_step for sz in m.batch_sizes)
    assert f.per_step[0].event_waits > 0


def test_virtual_polling_beats_fence_in_device_time(vstack):
    # the reference's modelled comparison (virtual clock, E=2 M=8, one
    # worker): polling keeps scheduling while a batch is open and fills it;
    # the fence blocks the only worker on the first request's probe, so
    # every batch launches alone
    p = vstack(workers=1, executors=2, max_agg=8).run(16, 1)
    f = vstack(workers=1, executors=2, max_agg=8, mode=IntegrationMode.FENCE).run(16, 1)
    assert p.checksum == f.checksum
    assert p.per_step[0].launches < f.per_step[0].launches
    assert p.per_step[0].wall_ms < f.per_step[0].wall_ms


def test_elided_barriers_ride_on_the_queue_tail():
    dev = VirtualClockDevice(barrier_elision=True, record_timeline=True)
    try:
        q = dev.queue()
        k = q.submit(make_kernel(100))
        b = q.submit(make_barrier())
        assert not b.is_complete()
        dev.advance_to_next()
        assert k.is_complete() and b.is_complete()
        assert [r[2] for r in dev.timeline] == ["kernel"]
        assert dev.snapshot_counters()["barriers_elided"] == 1
        b2 = q.submit(make_barrier())            # idle queue: completes at once
        assert b2.is_complete()
    finally:
        dev.destroy()


def test_interleaved_submission_order_matches_oracle():
    # the same per-queue programs submitted in another global order: the slot
    # goes to whichever kernel was submitted first, in both models alike
    per_q = {0: [s for s in SCRIPT if s[0] == 0], 1: [s for s in SCRIPT if s[0] == 1]}
    inter = [s for s in itertools.chain.from_iterable(
        itertools.zip_longest(per_q[1], per_q[0])) if s is not None]
    got, lat = run_script(inter, 1, 2)
    assert got == timeline(inter, lat, 1)
    assert got != run_script(SCRIPT, 1, 2)[0]
