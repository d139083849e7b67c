"""The command-line runner (reference cli.py / tests/test_cli.py behaviour).

Configuration resolution and exit codes run on CPU; full runs (which step the
CUDA path) are marked gpu and check the written diagnostics against the
reference's own PD trace (tests/golden/config1.npz, landau_pd2_trace).
"""

import csv
import json
from dataclasses import asdict

import numpy as np
import pytest

from conftest import golden

from paper_2605_10729_b200 import cli
from paper_2605_10729_b200.cli import EXIT_OK, EXIT_RUNTIME, EXIT_USAGE, RunConfig, main


def read_csv(path):
    with open(path) as f:
        return list(csv.DictReader(f))


# ---------------------------------------------------------------------------
# Configuration (CPU)
# ---------------------------------------------------------------------------

def test_paper_defaults():
    cfg = RunConfig(benchmark="landau").resolved()
    assert (cfg.dt, cfg.steps, cfg.eps_fine, cfg.modes, cfg.ppm) == (0.003125, 768, 1e-7, 16, 10)
    assert (cfg.strategy, cfg.shape, cfg.out_dir) == ("serial", "delta", "out")
    assert cfg.dt_coarse == 0.05 and cfg.blocks == 1 and cfg.coarse_modes == 16
    pic = RunConfig(benchmark="penning", coarse="pic").resolved()
    assert pic.blocks == 16 and pic.dt_coarse == pic.dt


@pytest.mark.parametrize("strategy", ["dd", "st"])
def test_out_of_scope_strategies_are_usage_errors(strategy, tmp_path):
    with pytest.raises(cli.UsageError):
        RunConfig(benchmark="landau", strategy=strategy).validate()
    assert main(["--benchmark", "landau", "--strategy", strategy, "--out-dir",
                 str(tmp_path / "x")]) == EXIT_USAGE
    assert not (tmp_path / "x").exists()


@pytest.mark.parametrize("argv", [
    ["--strategy", "pd"],                                         # no benchmark
    ["--benchmark", "landau", "--ranks-time", "2", "--strategy", "pd"],
    ["--benchmark", "landau", "--strategy", "serial", "--ranks-space", "2"],
    ["--benchmark", "landau", "--modes", "7"],
    ["--benchmark", "landau", "--steps", "0"],
    ["--benchmark", "landau", "--dt", "-1"],
])
def test_usage_errors_exit_2(argv, tmp_path):
    assert main(argv + ["--out-dir", str(tmp_path / "x")]) == EXIT_USAGE


def test_argparse_rejects_bad_choice():
    with pytest.raises(SystemExit) as ei:
        main(["--benchmark", "plasma"])
    assert ei.value.code == 2


def test_unknown_config_key_rejected(tmp_path):
    path = tmp_path / "cfg"
    path.write_text("benchmark=landau\nwibble=3\n")
    assert main(["--config", str(path)]) == EXIT_USAGE


def test_config_file_overlay_and_flag_override(tmp_path):
    path = tmp_path / "cfg"
    path.write_text("# desk run\nbenchmark=landau\nmodes=8\nppm=2\nsteps=4\ndt=0.05\n"
                    "log_comm=yes\n")
    cfg = cli.build_config(cli.make_parser().parse_args(["--config", str(path), "--steps", "6"]))
    assert (cfg.modes, cfg.ppm, cfg.steps, cfg.dt, cfg.log_comm) == (8, 2, 6, 0.05, True)


def test_json_config_file(tmp_path):
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps({"benchmark": "penning", "modes": 8, "strategy": "pd"}))
    cfg = cli.build_config(cli.make_parser().parse_args(["--config", str(path)]))
    assert (cfg.benchmark, cfg.modes, cfg.strategy) == ("penning", 8, "pd")


def test_presets_encode_desk_configs():
    for name, kind in (("desk-landau", "landau"), ("desk-penning", "penning")):
        cfg = cli.build_config(cli.make_parser().parse_args(["--preset", name]))
        assert (cfg.benchmark, cfg.modes, cfg.ppm, cfg.dt, cfg.steps) == (kind, 16, 10, 0.05, 100)


def test_every_config_field_has_a_flag():
    dests = {a.dest for a in cli.make_parser()._actions}
    assert {f for f in asdict(RunConfig(benchmark="landau"))} <= dests


# ---------------------------------------------------------------------------
# Full runs (GPU)
# ---------------------------------------------------------------------------

@pytest.mark.gpu
def test_pd_run_writes_reference_trace(tmp_path, capsys, cuda):
    out = tmp_path / "run"
    code = main(["--benchmark", "landau", "--strategy", "pd", "--modes", "16", "--ppm", "16",
                 "--dt", "0.05", "--steps", "20", "--ranks-space", "2", "--out-dir", str(out),
                 "--log-comm"])
    assert code == EXIT_OK
    rows = read_csv(out / "diagnostics.csv")
    assert [int(r["step"]) for r in rows] == list(range(1, 21))
    ref = golden("config1.npz")["landau_pd2_trace"][1:]
    for col, name in ((2, "field_energy"), (3, "kinetic_energy"), (4, "total_energy")):
        got = np.array([float(r[name]) for r in rows])
        assert np.max(np.abs(got - ref[:, col]) / np.abs(ref[:, col])) <= 1e-10, name
    meta = json.loads((out / "meta.json").read_text())
    assert meta["config"]["strategy"] == "pd"
    assert meta["rank_layout"] == {"space": 2, "time": 1, "total": 2}
    assert meta["initial_record"]["step"] == 0
    assert {r["rank"] for r in read_csv(out / "timers.csv")} == {"0", "1"}
    comm = read_csv(out / "comm_log.csv")
    assert {r["primitive"] for r in comm} == {"allreduce"}
    assert len(comm) == 2 * 21                  # one allreduce per step and rank
    assert "final_field_energy=" in capsys.readouterr().out


@pytest.mark.gpu
def test_meta_echoes_resolved_config(tmp_path, cuda):
    out = tmp_path / "run"
    cfg = cli.build_config(cli.make_parser().parse_args(
        ["--benchmark", "penning", "--modes", "8", "--ppm", "2", "--dt", "0.05", "--steps", "3",
         "--out-dir", str(out)]))
    assert cli.run(cfg) == EXIT_OK
    meta = json.loads((out / "meta.json").read_text())
    assert meta["config"] == asdict(cfg.resolved())
    assert len(read_csv(out / "diagnostics.csv")) == 3


@pytest.mark.gpu
def test_run_refuses_existing_outputs(tmp_path, cuda):
    argv = ["--benchmark", "landau", "--modes", "8", "--ppm", "2", "--dt", "0.05", "--steps", "2",
            "--out-dir", str(tmp_path / "dup")]
    assert main(argv) == EXIT_OK
    assert main(argv) == EXIT_RUNTIME
    assert main(argv + ["--overwrite"]) == EXIT_OK


def test_config_file_round_trip_property(tmp_path):
    """Any valid configuration written as key=value lines or JSON parses back to
    the same RunConfig (hypothesis)."""
    from hypothesis import given, settings
    from hypothesis import strategies as st

    cfgs = st.fixed_dictionaries({
        "benchmark": st.sampled_from(["landau", "penning"]),
        "strategy": st.sampled_from(["serial", "pd"]),
        "modes": st.integers(2, 40).map(lambda k: 2 * k),
        "ppm": st.integers(1, 64),
        "dt": st.floats(1e-4, 1.0),
        "steps": st.integers(1, 1000),
        "eps_fine": st.sampled_from([1e-3, 1e-7, 1e-12]),
        "shape": st.sampled_from(["delta", "cic"]),
        "seed": st.integers(0, 2 ** 31),
        "log_comm": st.booleans(),
    })

    @settings(max_examples=60, deadline=None)
    @given(cfgs, st.booleans())
    def check(d, as_json):
        path = tmp_path / ("c.json" if as_json else "c.txt")
        if as_json:
            path.write_text(json.dumps(d))
        else:
            path.write_text("\n".join(f"{k} = {v!r}" if isinstance(v, float) else f"{k}={v}"
                                      for k, v in d.items()))
        cfg = cli.build_config(cli.make_parser().parse_args(["--config", str(path)]))
        for k, v in d.items():
            assert getattr(cfg, k) == v, (k, getattr(cfg, k), v)

    check()
