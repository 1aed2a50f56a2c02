"""benchcli contract on CPU: flags, exit codes, sweep layouts, CSV/JSON rows
(pkg/tests/test_cli.py); the GPU run itself is tests/test_gpu_ablation.py."""

import json

import pytest

from paper_2303_08058_b200 import cli
from paper_2303_08058_b200.bridge import IntegrationMode


def test_defaults_match_reference():
    cfg = cli.config_from_args(cli.parse_args([]))
    assert (cfg.workers, cfg.executors, cfg.max_agg, cfg.subgrids, cfg.steps) == \
        (8, 32, 8, 64, 15)
    assert cfg.integration is IntegrationMode.POLLING and cfg.repeats == 3


@pytest.mark.parametrize("argv", [["--workers", "0"], ["--executors", "x"],
                                  ["--integration", "magic"], ["--clock", "sundial"],
                                  ["--watchdog", "-1"], ["--nope"]])
def test_usage_errors_exit_1(argv):
    with pytest.raises(SystemExit) as e:
        cli.parse_args(argv)
    assert e.value.code == cli.EXIT_USAGE


def test_sweep_layouts():
    base = cli.RunConfig()
    ex = cli.sweep_cells(base, "executors")
    assert [c.executors for c in ex] == [1, 2, 4, 8, 16, 32, 64, 128]
    assert {c.max_agg for c in ex} == {1}
    ag = cli.sweep_cells(base, "aggregation")
    assert [c.max_agg for c in ag] == [1, 2, 4, 8, 16, 32, 64] and {c.executors for c in ag} == {1}
    assert [c.workers for c in cli.sweep_cells(base, "workers")] == [1, 2, 4, 8]
    assert cli.sweep_cells(base, "none") == [base]


def _fake_cell(cfg, ms, checksum=1.5):
    return cli.CellResult(cfg=cfg, mean_step_ms=ms, stddev_ms=0.1, launches=10,
                          mean_batch=2.0, checksum=checksum)


def test_matrix_adds_fence_twin_and_formats(monkeypatch, tmp_path):
    def fake_run_cell(cfg, devices=None):
        return _fake_cell(cfg, 10.0 if cfg.integration is IntegrationMode.FENCE else 5.0)

    monkeypatch.setattr(cli, "run_cell", fake_run_cell)
    rows, failures = cli.run_matrix([cli.RunConfig(), cli.RunConfig(
        integration=IntegrationMode.FENCE)])
    assert not failures and len(rows) == 2
    by_mode = {r["mode"]: r for r in rows}
    assert by_mode["polling"]["speedup_vs_fence"] == 2.0
    assert by_mode["fence"]["speedup_vs_fence"] == 1.0
    text = cli.format_csv(rows)
    assert text.splitlines()[0] == ",".join(cli.CSV_COLUMNS)
    assert text.splitlines()[1].startswith("8,32,8,fence,off,10.000000")
    js = json.loads(cli.format_json(rows))
    assert [r["mode"] for r in js] == ["fence", "polling"]
    assert js[0]["checksum"] == float.hex(1.5)
    out = tmp_path / "o.csv"
    cli.emit(rows, "csv", str(out))
    assert out.read_text() == text


def test_exit_codes(monkeypatch, tmp_path):
    monkeypatch.setattr(cli, "run_cell", lambda cfg, devices=None: _fake_cell(cfg, 1.0))
    assert cli.main(["--out", str(tmp_path / "a.csv")]) == cli.EXIT_OK

    def boom(cfg, devices=None):
        raise RuntimeError("cell died")

    monkeypatch.setattr(cli, "run_cell", boom)
    assert cli.main(["--out", str(tmp_path / "b.csv")]) == cli.EXIT_RUN_FAILED

    monkeypatch.setattr(cli, "run_cell", lambda cfg, devices=None: _fake_cell(cfg, 1.0, float(cfg.workers)))
    assert cli.main(["--sweep", "workers", "--out", str(tmp_path / "c.csv")]) == \
        cli.EXIT_CHECKSUM

    def interrupt(cfg, devices=None):
        raise KeyboardInterrupt

    monkeypatch.setattr(cli, "run_cell", interrupt)
    assert cli.main(["--out", str(tmp_path / "d.csv")]) == cli.EXIT_INTERRUPTED
    monkeypatch.setattr(cli, "run_cell", lambda cfg, devices=None: _fake_cell(cfg, 1.0))
    assert cli.main(["--out", str(tmp_path / "no" / "such" / "dir.csv")]) == \
        cli.EXIT_RUN_FAILED


def test_virtual_clock_without_simulator_is_a_usage_error(tmp_path):
    # the CUDA device runs on the real clock; --clock virtual needs the
    # simulator double injected (tests/test_virtual_clock.py)
    assert cli.main(["--clock", "virtual", "--out", str(tmp_path / "v.csv")]) == cli.EXIT_USAGE
