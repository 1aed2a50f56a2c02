"""The native machine on the hydro kernel (the paper's Octo-Tiger experiment
shape: per-sub-grid hydro tasks, aggregated launches,
polling vs host-task vs fence): bit-identical to the self-authored oracle's
forward-Euler steps (PARITY UNPINNED against the reference, which has no
hydro) in every completion mode and aggregation width."""

import math

import numpy as np
import pytest

from oracle import hydro_oracle as h

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["polling", "hosttask", "fence"])
@pytest.mark.parametrize("max_agg,task_subgrids", [(1, 1), (4, 1), (8, 2)])
def test_hydro_machine_matches_oracle(mode, max_agg, task_subgrids):
    from paper_2303_08058_b200.bridge import IntegrationMode
    from paper_2303_08058_b200.native_machine import run_native_hydro
    I, _ = h.rotating_star(27)
    steps, dts = 2, []
    want = I
    for _ in range(steps):
        want, dt = h.euler_step(want)
        dts.append(dt)
    per_step, got = run_native_hydro(I, steps, workers=4, executors=3, max_agg=max_agg,
                                     mode=IntegrationMode(mode), task_subgrids=task_subgrids)
    assert np.array_equal(got, want)
    assert [m.dt for m in per_step] == dts
    assert per_step[-1].checksum_piece == math.fsum(want[:, 0].ravel().tolist())
    assert per_step[0].launches >= 27 // (max_agg * task_subgrids)


def test_hydro_machine_aggregates_under_polling():
    from paper_2303_08058_b200.bridge import IntegrationMode
    from paper_2303_08058_b200.native_machine import run_native_hydro
    I, _ = h.rotating_star(512)
    per_step, _ = run_native_hydro(I, 2, workers=8, executors=8, max_agg=8,
                                   mode=IntegrationMode.POLLING)
    for m in per_step:
        assert m.launches <= 512 and m.reasons_full + m.reasons_idle == m.launches
        assert m.event_waits == 0
    per_fence, _ = run_native_hydro(I, 1, workers=8, executors=8, max_agg=8,
                                    mode=IntegrationMode.FENCE)
    assert per_fence[0].event_waits > 0
