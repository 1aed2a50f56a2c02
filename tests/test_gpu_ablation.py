"""Acceptance on a B200: event polling beats fencing (the paper's claim,
PAPER.md:1049-1054; reference criterion 3, pkg/tests/test_acceptance.py:80-91)
and the checksum is identical across modes (criterion 2). Directional
timing assertions only, with the reference's own margin."""

import pytest

from conftest import fx

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")


def test_criterion3_polling_beats_fence_on_gpu(golden):
    from paper_2303_08058_b200.bridge import IntegrationMode
    from paper_2303_08058_b200.cli import RunConfig, run_cell
    from dataclasses import replace
    base = RunConfig(subgrids=64, steps=15, repeats=3, executors=1, max_agg=8, workers=4)
    polling = run_cell(replace(base, integration=IntegrationMode.POLLING))
    fence = run_cell(replace(base, integration=IntegrationMode.FENCE))
    speedup = fence.mean_step_ms / polling.mean_step_ms
    print(f"polling {polling.mean_step_ms:.3f} ms/step vs fence {fence.mean_step_ms:.3f}"
          f" -> speedup {speedup:.3f}")
    assert polling.checksum == fence.checksum
    assert speedup >= 1.05


def test_paper_scenario_512_polling_vs_fence():
    # 512 sub-grids, 32 executors x max 8 aggregated
    from paper_2303_08058_b200.bridge import IntegrationMode
    from paper_2303_08058_b200.cli import RunConfig, run_matrix
    # 4 workers: the paper's best combination on a weakened CPU (its third
    # graph); at 8 of the box's 16 cores the two modes are within a few %
    # (1.03-1.09x, profiles/r02/bench_session4*.json), too close to assert
    rows, failures = run_matrix([RunConfig(subgrids=512, steps=4, repeats=3, executors=32,
                                           max_agg=8, workers=4,
                                           integration=IntegrationMode.POLLING)])
    assert not failures
    print(rows[0])
    assert rows[0]["speedup_vs_fence"] >= 1.05


# Criteria 4 and 5 (pkg/tests/test_acceptance.py:94-122) on the reference-API
# path, which run_scenario delegates to the native machine (engine "native"
# in the CLI): measured 1.8-2.0x and 1.16x on a B200
# (profiles/r02/criteria45.jsonl). The GIL-bound Python machine is timed there
# too (1.03-1.06x; elision 0.95-1.00x, as the reference's own 8-core run of
# criterion 5, pkg/test_output.txt:152) but not asserted.
def test_criterion4_hosttask_no_faster_than_polling_on_gpu():
    from dataclasses import replace

    from paper_2303_08058_b200.bridge import IntegrationMode
    from paper_2303_08058_b200.cli import RunConfig, run_cell
    base = RunConfig(subgrids=64, steps=15, repeats=3, executors=1, max_agg=32, workers=8,
                     engine="native")
    hosttask = run_cell(replace(base, integration=IntegrationMode.HOSTTASK))
    polling = run_cell(replace(base, integration=IntegrationMode.POLLING))
    ratio = hosttask.mean_step_ms / polling.mean_step_ms
    print(f"hosttask {hosttask.mean_step_ms:.3f} vs polling {polling.mean_step_ms:.3f} "
          f"-> {ratio:.3f}")
    assert hosttask.checksum == polling.checksum
    assert ratio >= 1.0


def test_criterion5_barrier_elision_helps_on_gpu():
    from dataclasses import replace

    from paper_2303_08058_b200.bridge import IntegrationMode
    from paper_2303_08058_b200.cli import RunConfig, run_cell
    base = RunConfig(subgrids=64, steps=15, repeats=3, executors=1, max_agg=2, workers=4,
                     integration=IntegrationMode.POLLING, inject_barriers=True,
                     engine="native")
    on = run_cell(replace(base, barrier_elision=True))
    off = run_cell(replace(base, barrier_elision=False))
    ratio = off.mean_step_ms / on.mean_step_ms
    print(f"elision on {on.mean_step_ms:.3f} vs off {off.mean_step_ms:.3f} -> {ratio:.3f}")
    assert on.checksum == off.checksum
    assert ratio > 1.0
