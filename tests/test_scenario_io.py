"""Scenario text/binary formats and trajectory dumps (paper_0911_2900_b200/scenario_io.py,
SURVEY §8f rows 3-4): the text grammar against the reference's own cases
(tests/test_world.cpp:37-125), binary and trajectory round trips, and -- on the GPU -- a recorded
device trajectory against the reference engine step by step."""
import os

import numpy as np
import pytest

import oracle
from paper_0911_2900_b200 import fastped as fp
from paper_0911_2900_b200 import scenario_io as sio
from tests.helpers import random_grid

TINY = "FAST-SCENARIO v1\nwidth 3\nheight 3\ncell_size 0.4\nboundary closed\ngrid:\n###\n#E#\n###\n"


def test_parse_smallest_legal_grid():
    g = sio.parse_scenario(TINY)
    assert (g.width, g.height, g.cell_size, g.boundary) == (3, 3, 0.4, fp.CLOSED)
    assert g.cells[1, 1] == fp.EXIT and g.exit_cell_count() == 1 and g.free_cell_count() == 0


def test_unknown_cell_character_reports_its_line():
    i = TINY.find("E", TINY.find("grid:"))
    with pytest.raises(RuntimeError, match=r"line 8: unknown cell character 'X'"):
        sio.parse_scenario(TINY[:i] + "X" + TINY[i + 1:])


def test_periodic_corridor_round_trip():
    text = ("FAST-SCENARIO v1\nwidth 5\nheight 4\ncell_size 0.4\nboundary periodic-x\ngrid:\n"
            "#####\n.....\n.....\n#####\n")
    g = sio.parse_scenario(text)
    assert (g.boundary, g.width, g.height, g.free_cell_count()) == (fp.PERIODIC_X, 5, 4, 10)
    assert sio.serialize_scenario(g) == text


def test_structural_errors_carry_line_numbers():
    with pytest.raises(RuntimeError, match="line 1.*malformed header"):
        sio.parse_scenario("FAST-SCENARIO v2\n")
    with pytest.raises(RuntimeError, match="line 2"):
        sio.parse_scenario("FAST-SCENARIO v1\nwidth x\n")
    with pytest.raises(RuntimeError, match="line 8.*dimension mismatch|dimension mismatch.*"):
        sio.parse_scenario(TINY.replace("#E#", "#E"))
    with pytest.raises(RuntimeError, match="dimension mismatch"):
        sio.parse_scenario(TINY[:TINY.rfind("###")])
    with pytest.raises(RuntimeError, match="line 7: closed boundary violated"):
        sio.parse_scenario(TINY.replace("###", "#.#", 1))
    with pytest.raises(RuntimeError, match="unexpected content"):
        sio.parse_scenario(TINY + "##\n")
    with pytest.raises(RuntimeError, match="periodic-x boundary violated"):
        sio.parse_scenario("FAST-SCENARIO v1\nwidth 4\nheight 3\ncell_size 0.4\nboundary periodic-x\ngrid:\n"
                           "##.#\n....\n####\n")


def test_parse_after_serialize_is_identity_on_random_grids(tmp_path):
    rng = np.random.default_rng(2024)
    for i in range(40):
        g = fp.Grid(random_grid(rng, int(rng.integers(3, 25)), int(rng.integers(3, 25)), 0.2, 2))
        assert np.array_equal(sio.parse_scenario(sio.serialize_scenario(g)).cells, g.cells)
    p = tmp_path / "plaza.txt"
    sio.save_scenario(fp.make_plaza(8.0, 2), str(p))
    assert sio.parse_scenario(p.read_text()).free_cell_count() == 324


def test_binary_scenario_round_trip(tmp_path):
    rng = np.random.default_rng(7)
    g = fp.Grid(random_grid(rng, 37, 21, 0.15, 3), 0.5)
    field = rng.random(g.cells.shape)
    p = str(tmp_path / "g.fsb")
    sio.save_scenario_binary(fp.Scenario("g", g, field), p)
    sc = sio.load_scenario_binary(p)
    assert sc.name == "g.fsb" and sc.grid.cell_size == 0.5 and sc.grid.boundary == fp.CLOSED
    assert np.array_equal(sc.grid.cells, g.cells) and np.array_equal(sc.field, field)
    with open(p, "r+b") as f:
        f.write(b"NOTMAGIC")
    with pytest.raises(RuntimeError, match="bad magic"):
        sio.load_scenario_binary(p)


def test_trajectory_file_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    n, w, h = 37, 9, 5
    frames = [sio.StepSnapshot(s, rng.integers(0, w, n).astype(np.int32), rng.integers(0, h, n).astype(np.int32),
                               rng.random(n) < 0.8, rng.permutation(n)[: s].astype(np.uint32),
                               rng.integers(-1, n, (h, w)).astype(np.int32)) for s in range(1, 6)]
    p = str(tmp_path / "t.trj")
    with sio.TrajectoryWriter(p, n, w, h, with_occupancy=True) as tw:
        for f in frames:
            tw.write(f)
    assert list(sio.read_trajectory(p)) == frames


@pytest.mark.gpu
def test_load_scenario_computes_the_reference_field(tmp_path):
    rng = np.random.default_rng(11)
    g = fp.Grid(random_grid(rng, 40, 30, 0.2, 3))
    p = str(tmp_path / "s.txt")
    sio.save_scenario(g, p)
    sc = sio.load_scenario(p)
    assert sc.name == "s.txt"
    assert np.array_equal(sc.field, oracle.ref_static_field(g.cells).reshape(sc.field.shape))
    sio.save_scenario_binary(g, str(tmp_path / "s.fsb"), with_field=False)
    assert np.array_equal(sio.load_scenario_binary(str(tmp_path / "s.fsb")).field, sc.field)


@pytest.mark.gpu
def test_recorded_trajectory_matches_the_reference(tmp_path):
    sc = fp.make_scenario("plaza", fp.make_plaza(12.0, 3))
    params = fp.SimParams(k_s=1.2, v_max=4, seed=0xACCE55, steps=20)
    p = str(tmp_path / "run.trj")
    traj = sio.record_trajectory(sc, 200, params, 4, 20, p, with_occupancy=True)
    assert list(sio.read_trajectory(p)) == traj
    r = fp.spawn_agents(sc.grid, 200, 4, params.seed)
    ref = oracle.RefState(sc.grid.cells, sc.field, r.x, r.y, 4)
    for snap in traj:
        ex, _ = ref.step_once(params.k_s, params.seed)
        x, y, a = ref.agents()
        assert np.array_equal(snap.x, x) and np.array_equal(snap.y, y)
        assert np.array_equal(snap.alive, a.astype(bool)) and np.array_equal(snap.exited, ex)
        assert np.array_equal(snap.occupancy, ref.occupancy().reshape(snap.occupancy.shape))
