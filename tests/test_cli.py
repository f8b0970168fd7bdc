"""The command-line harness (paper_0911_2900_b200/cli.py), mirroring the reference's
tools/fastped.cpp: option surface and error exits on CPU; on the GPU, each engine subcommand's
files against the library calls (and the fundamental diagram against the compiled reference)."""
import numpy as np
import pytest

import oracle
from paper_0911_2900_b200 import cli
from paper_0911_2900_b200 import fastped as fp
from paper_0911_2900_b200 import harness as hz
from paper_0911_2900_b200 import scenario_io as sio
from paper_0911_2900_b200 import scenarios


def run_cli(argv, capsys):
    rc = cli.main([str(a) for a in argv])
    out = capsys.readouterr()
    return rc, out.out, out.err


# ---------------------------------------------------------------- host-only subcommands
def test_speedup_matches_harness(tmp_path, capsys):
    recs = [hz.RunRecord("plaza", 1000, 4, 1, 396, 2.0, 1.5, 0.5, 1),
            hz.RunRecord("plaza", 1000, 4, 2, 396, 1.0, 0.75, 0.25, 1),
            hz.RunRecord("plaza", 1000, 4, 8, 396, 0.4, 0.3, 0.1, 1)]
    src = tmp_path / "sweep.csv"
    src.write_text(hz.runs_to_csv(recs))
    dst = tmp_path / "speedup.csv"
    rc, out, _ = run_cli(["speedup", "--in", src, "--out", dst], capsys)
    assert rc == 0
    assert dst.read_text() == hz.speedups_to_csv(hz.speed_factor(recs))
    assert "5.000" in out and "wrote " + str(dst) in out


def test_speedup_without_baseline_is_an_error(tmp_path, capsys):
    src = tmp_path / "sweep.csv"
    src.write_text(hz.runs_to_csv([hz.RunRecord("plaza", 10, 4, 2, 5, 1.0, 0.5, 0.5, 1)]))
    rc, _, err = run_cli(["speedup", "--in", src, "--out", tmp_path / "o.csv"], capsys)
    assert rc == 1 and err.startswith("fastped: speed_factor: no 1-core baseline")


@pytest.mark.parametrize("config", ["corridor", "room", "ring"])
def test_scenario_text_round_trip(tmp_path, capsys, config):
    path = tmp_path / (config + ".txt")
    rc, out, _ = run_cli(["scenario", "--config", config, "--out", path], capsys)
    assert rc == 0 and str(path) in out
    g = sio.parse_scenario(path.read_text())
    ref = scenarios.build(config, n=0).grid
    assert (g.width, g.height, g.boundary) == (ref.width, ref.height, ref.boundary)
    np.testing.assert_array_equal(g.cells, ref.cells)


def test_scenario_binary_geometry(tmp_path, capsys):
    path = tmp_path / "obst.fscb"
    rc, _, _ = run_cli(["scenario", "--config", "obstacles", "--width", 300, "--height", 80, "--seed", 5,
                        "--out", path], capsys)
    assert rc == 0
    assert path.read_bytes()[:8] == sio.BINARY_MAGIC
    ref = scenarios.obstacles(seed=5, n=0, width=300, height=80).grid
    with open(path, "rb") as f:
        f.seek(sio._BIN_HEAD.size)
        cells = np.fromfile(f, np.uint8)
    np.testing.assert_array_equal(cells.reshape(80, 300), ref.cells)


def test_usage_errors_exit_2(capsys):
    with pytest.raises(SystemExit) as e:
        cli.main(["fd", "--out", "x.csv"])  # --densities is required (tools/fastped.cpp:191-194)
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main([])  # app.require_subcommand(1)
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["sweep", "--scenario", "s", "--agents", "1,x", "--out", "o"])
    assert e.value.code == 2
    capsys.readouterr()


def test_runtime_errors_exit_1(tmp_path, capsys):
    rc, _, err = run_cli(["run", "--scenario", tmp_path / "missing.txt", "--agents", 5, "--out",
                          tmp_path / "o.csv"], capsys)
    assert rc == 1 and err.startswith("fastped: cannot open scenario file")
    rc, _, err = run_cli(["scenario", "--config", "room", "--width", 50, "--out", tmp_path / "r.txt"], capsys)
    assert rc == 1 and "plaza and obstacles only" in err


def test_defaults_follow_the_reference():
    p = cli.build_parser()
    a = p.parse_args(["run", "--scenario", "s", "--agents", "3", "--out", "o"])
    assert (a.vmax, a.cores, a.steps, a.seed) == (4, 1, 396, 1)
    a = p.parse_args(["sweep", "--scenario", "s", "--agents", "10,20", "--out", "o"])
    assert (a.cores, a.agents, a.vmax, a.reps) == ([1, 2, 4, 8], [10, 20], [4], 3)
    a = p.parse_args(["realtime", "--scenario", "s", "--out", "o"])
    assert (a.budget_steps, a.dt, a.start_n) == (396, 1.0, 1000)
    a = p.parse_args(["fd", "--densities", "0.5,1", "--out", "o"])
    assert (a.length_m, a.width_m, a.warmup, a.measure, a.drive_gradient, a.cell_size) == \
        (50.0, 4.0, 100, 296, 8.0, 0.4)
    assert a.densities == [0.5, 1.0]
    assert p.parse_args(["run", "--scenario", "s", "--agents", "3", "--out", "o", "--seed", "0xACCE55"]).seed == \
        0xACCE55


# ---------------------------------------------------------------- engine subcommands (GPU)
@pytest.fixture
def plaza_file(tmp_path):
    path = tmp_path / "mini.txt"
    sio.save_scenario(fp.make_plaza(8.0, 2), str(path))  # 20x20
    return path


@pytest.mark.gpu
def test_cli_run_matches_library(tmp_path, capsys, plaza_file):
    out_csv = tmp_path / "run.csv"
    rc, out, _ = run_cli(["run", "--scenario", plaza_file, "--agents", 150, "--steps", 40, "--seed", 3,
                          "--out", out_csv], capsys)
    assert rc == 0
    rec, = hz.parse_run_csv(out_csv.read_text())
    assert (rec.scenario, rec.agents_initial, rec.v_max, rec.cores, rec.steps, rec.seed) == \
        ("mini.txt", 150, 4, 1, 40, 3)
    sc = sio.load_scenario(str(plaza_file))
    st = fp.make_state(sc, fp.spawn_agents(sc.grid, 150, 4, 3))
    rs = fp.run(st, fp.SimParams(seed=3, steps=40))
    st.close()
    assert "exited %d, alive %d" % (rs.exited, rs.alive) in out


@pytest.mark.gpu
def test_cli_fd_matches_reference(tmp_path, capsys):
    out_csv = tmp_path / "fd.csv"
    rc, out, _ = run_cli(["fd", "--length-m", 10, "--width-m", 2, "--densities", "0.5,1,2,4", "--seed", 9,
                          "--warmup", 50, "--measure", 120, "--out", out_csv], capsys)
    assert rc == 0 and "weidmann_ref" in out
    corridor = fp.make_corridor(10.0, 2.0)
    d, s, f = oracle.ref_fundamental_diagram(corridor.cells, corridor.cell_size, 4, [0.5, 1.0, 2.0, 4.0], 9, 50, 120)
    assert out_csv.read_text() == hz.fd_to_csv([hz.FdRecord(*r) for r in zip(d, s, f)])


@pytest.mark.gpu
def test_cli_realtime_and_sweep(tmp_path, capsys, plaza_file):
    cap_csv = tmp_path / "cap.csv"
    rc, out, _ = run_cli(["realtime", "--scenario", plaza_file, "--budget-steps", 3, "--start-n", 10,
                          "--out", cap_csv], capsys)
    assert rc == 0 and "ran out of free cells" in out
    head, row = cap_csv.read_text().splitlines()
    assert head.startswith("scenario,v_max,cores,budget_steps")
    f = row.split(",")
    assert f[0] == "mini.txt" and int(f[5]) == 324
    sweep_csv = tmp_path / "sweep.csv"
    rc, out, _ = run_cli(["sweep", "--scenario", plaza_file, "--cores", "1,2", "--agents", "5,20", "--vmax", "2,4",
                          "--steps", 5, "--reps", 1, "--out", sweep_csv], capsys)
    assert rc == 0 and out.startswith("8 records")
    recs = hz.parse_run_csv(sweep_csv.read_text())
    assert [(r.agents_initial, r.v_max, r.cores) for r in recs] == \
        [(a, v, c) for a in (5, 20) for v in (2, 4) for c in (1, 2)]


@pytest.mark.gpu
def test_cli_trajectory_matches_record_trajectory(tmp_path, capsys, plaza_file):
    path = tmp_path / "t.trj"
    rc, _, _ = run_cli(["trajectory", "--scenario", plaza_file, "--agents", 120, "--steps", 12, "--occupancy",
                        "--out", path], capsys)
    assert rc == 0
    got = list(sio.read_trajectory(str(path)))
    sc = sio.load_scenario(str(plaza_file))
    want = sio.record_trajectory(sc, 120, fp.SimParams(seed=1, steps=12), 1, 12, with_occupancy=True)
    assert len(got) == 12 and got == want
