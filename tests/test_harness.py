"""The measurement harness (paper_0911_2900_b200/harness.py) against the
reference's own known answers (tests/test_bench.cpp, tests/test_scenario_io.cpp) and against
the compiled reference (oracle/_ref): capacity search on timing tables, and -- on the GPU -- the
fundamental diagram bit for bit."""
import math

import numpy as np
import pytest

import oracle
from paper_0911_2900_b200 import fastped as fp
from paper_0911_2900_b200 import harness as hz


# ---------------------------------------------------------------- Weidmann (test_bench.cpp:162-178)
def test_weidmann_closed_form():
    assert hz.weidmann_speed(0.0) == 1.34
    assert hz.weidmann_speed(5.4) == 0.0
    assert hz.weidmann_speed(6.0) == 0.0
    assert hz.weidmann_speed(1.0) == pytest.approx(1.0580628560768004, abs=1e-9)
    assert hz.weidmann_speed(0.5) == pytest.approx(1.298375699131641, abs=1e-9)
    assert hz.weidmann_speed(3.0) == pytest.approx(0.330694766470473, abs=1e-9)
    with pytest.raises(ValueError):
        hz.weidmann_speed(-0.1)


def test_compare_weidmann_reports_absolute_errors():
    rows = hz.compare_weidmann([hz.FdRecord(1.0, 1.0, 1.0)])
    assert len(rows) == 1
    assert rows[0].reference_speed == pytest.approx(1.0580628560768004, abs=1e-9)
    assert rows[0].abs_error == pytest.approx(0.0580628560768004, abs=1e-9)


# ---------------------------------------------------------------- speed factors (test_bench.cpp:46-83)
def test_sweep_spec_validation():
    spec = hz.SweepSpec()
    with pytest.raises(ValueError):
        spec.validate()
    spec = hz.SweepSpec([1], [10], [4])
    spec.validate()
    for bad in (hz.SweepSpec([0], [10], [4]), hz.SweepSpec([1], [0], [4]), hz.SweepSpec([1], [10], [6]),
                hz.SweepSpec([1], [10], [4], steps=0), hz.SweepSpec([1], [10], [4], repetitions=0)):
        with pytest.raises(ValueError):
            bad.validate()


def test_speed_factor_ideal_timings():
    recs = [hz.RunRecord("syn", 1000, 4, c, 1, 8.0 / c, 0, 0, 1) for c in (1, 2, 4, 8)]
    rows = hz.speed_factor(recs)
    assert [r.factor for r in rows] == [1.0, 2.0, 4.0, 8.0]


def test_speed_factor_needs_a_one_core_baseline():
    with pytest.raises(RuntimeError, match="no 1-core baseline.*agents=1000"):
        hz.speed_factor([hz.RunRecord("syn", 1000, 4, 2, 1, 4.0, 0, 0, 1)])


def test_speedup_csv_three_decimals():
    assert hz.speedups_to_csv([hz.SpeedupRow("syn", 10, 4, 2, 0.5, 1.23456)]) == (
        "scenario,agents_initial,v_max,cores,wall_time_s,factor\nsyn,10,4,2,0.500000,1.235\n")


# ---------------------------------------------------------------- run CSV (test_scenario_io.cpp:93-115)
def test_run_csv_is_byte_exact_and_round_trips():
    assert hz.runs_to_csv([]) == hz.RUN_CSV_HEADER + "\n"
    rec = hz.RunRecord("plaza", 1000, 4, 8, 396, 1.5, 1.25, 0.125, 42)
    text = hz.runs_to_csv([rec])
    assert text == hz.RUN_CSV_HEADER + "\nplaza,1000,4,8,396,1.500000,1.250000,0.125000,42\n"
    assert "\n\n" not in text
    recs = [hz.RunRecord("plaza84", 40000, 4, 1, 50, 12.345678, 11.5, 0.25, 7),
            hz.RunRecord("plaza84", 40000, 4, 8, 50, 3.000001, 2.75, 0.25, 7),
            hz.RunRecord("corridor", 123, 1, 2, 396, 0.000002, 0.000001, 0.000001, 99)]
    assert hz.parse_run_csv(hz.runs_to_csv(recs)) == recs
    with pytest.raises(RuntimeError, match="header"):
        hz.parse_run_csv("nope\n")
    with pytest.raises(ValueError):
        hz.runs_to_csv([hz.RunRecord("a,b")])


def test_fd_csv():
    assert hz.fd_to_csv([hz.FdRecord(0.5, 1.6, 0.8)]) == "density,mean_speed,flow\n0.500000,1.600000,0.800000\n"


# ---------------------------------------------------------------- capacity (test_bench.cpp:85-120)
def _table(fn, start=1000, max_n=(2 ** 63 - 1) // 2, budget=396.0):
    """Every probe the doubling search can make, with its timing."""
    ns, n = [], start
    while True:
        ns.append(n)
        if fn(n) > budget or n >= max_n:
            break
        n = min(2 * n, max_n)
    return ns, [fn(k) for k in ns]


@pytest.mark.parametrize("fn,max_n", [
    (lambda n: 0.002 * n, (2 ** 63 - 1) // 2),      # linear: exact interpolation
    (lambda n: 1.0 * n, (2 ** 63 - 1) // 2),        # budget exceeded at the start
    (lambda n: 1e-6 * float(n) ** 1.3, (2 ** 63 - 1) // 2),
    (lambda n: 1e-9 * n, 5000),                      # scenario cap
    (lambda n: 3e-4 * n + 17.5, (2 ** 63 - 1) // 2),
])
def test_realtime_capacity_matches_reference(fn, max_n):
    res = hz.realtime_capacity(fn, 396.0, 1000, max_n)
    if oracle.have_reference():
        ns, ts = _table(fn, max_n=max_n)
        ref = oracle.ref_capacity_from_table(ns, ts, 396.0, 1000, max_n)
        for k in ("capacity", "n_low", "n_high", "below_start", "capped", "t_low_s", "t_high_s", "budget_s"):
            assert getattr(res, k) == ref[k], k


def test_realtime_capacity_known_answers():
    r = hz.realtime_capacity(lambda n: 0.002 * n, 396.0)
    assert (r.capacity, r.n_low, r.n_high, r.below_start, r.capped) == (198000, 128000, 256000, False, False)
    r = hz.realtime_capacity(lambda n: 1.0 * n, 396.0)
    assert r.below_start and r.n_high == 1000 and r.t_high_s == 1000.0 and r.capacity == -1
    timing = lambda n: 1e-6 * float(n) ** 1.3  # noqa: E731
    r = hz.realtime_capacity(timing, 396.0)
    assert r.t_low_s <= 396.0 < r.t_high_s and r.n_high == 2 * r.n_low and r.n_low <= r.capacity < r.n_high
    assert timing(r.capacity) <= 396.0 + 1e-6
    r = hz.realtime_capacity(lambda n: 1e-9 * n, 396.0, 1000, 5000)
    assert r.capped and r.capacity == 5000
    for args in ((0.0,), (1.0, 0), (1.0, 10, 5)):
        with pytest.raises(ValueError):
            hz.realtime_capacity(lambda n: 1.0, *args)


# ---------------------------------------------------------------- sweep / FD validation (host side)
def test_run_sweep_checks_capacity_before_timing():
    g = fp.make_plaza(4.0, 2)
    sc = fp.Scenario("mini", g, np.zeros(g.cells.shape))
    with pytest.raises(RuntimeError, match="has capacity %d but the sweep asks for 1000 agents" % g.free_cell_count()):
        hz.run_sweep(hz.SweepSpec([1], [1000], [4], steps=5, repetitions=1), sc, 1)


def test_fundamental_diagram_rejects_anything_but_a_sealed_periodic_corridor():
    with pytest.raises(ValueError):
        hz.fundamental_diagram(fp.make_plaza(4.0, 1), 4, [1.0], 1)
    corridor = fp.make_corridor(10.0, 2.0)
    with pytest.raises(ValueError):
        hz.fundamental_diagram(corridor, 4, [1.0], 1, -1, 10)
    with pytest.raises(ValueError):
        hz.fundamental_diagram(corridor, 4, [1.0], 1, 0, 0)
    with pytest.raises(RuntimeError, match="exceeds the capacity"):
        hz.fundamental_diagram(corridor, 4, [7.0], 1)
    with pytest.raises(ValueError, match="zero agents"):
        hz.fundamental_diagram(corridor, 4, [0.0], 1)


# ---------------------------------------------------------------- device runs
@pytest.mark.gpu
@pytest.mark.parametrize("length,width,densities,seed,warmup,measure", [
    (10.0, 2.0, [0.5, 1.0, 2.0, 4.0], 9, 50, 120),         # test_bench.cpp:154-160
    (40.0, 4.0, [0.25, 1.5, 3.0, 5.5], 20250811, 30, 60),
    (60.0, 2.4, [2.0], 7, 0, 25),
])
def test_fundamental_diagram_matches_reference(length, width, densities, seed, warmup, measure):
    corridor = fp.make_corridor(length, width)
    fd = hz.fundamental_diagram(corridor, 4, densities, seed, warmup, measure)
    d, s, f = oracle.ref_fundamental_diagram(corridor.cells, corridor.cell_size, 4, densities, seed, warmup, measure)
    assert [r.density for r in fd] == list(d)
    assert [r.mean_speed for r in fd] == list(s)
    assert [r.flow for r in fd] == list(f)


@pytest.mark.gpu
def test_fundamental_diagram_free_flow_and_saturation():
    corridor = fp.make_corridor(10.0, 2.0)  # 25x5: 75 free cells, 12 m^2
    rho_one = 1.0 / (corridor.free_cell_count() * 0.4 * 0.4)
    fd = hz.fundamental_diagram(corridor, 4, [rho_one], 20250811)
    assert fd[0].mean_speed == pytest.approx(1.6, abs=0.01)
    assert fd[0].flow == pytest.approx(fd[0].density * fd[0].mean_speed, abs=1e-9)
    fd = hz.fundamental_diagram(corridor, 4, [1.0 / (0.4 * 0.4)], 3, 10, 20)
    assert fd[0].mean_speed == 0.0 and fd[0].flow == 0.0
    fd = hz.fundamental_diagram(corridor, 4, [0.5, 1.0, 2.0, 4.0], 9, 50, 120)
    for a, b in zip(fd, fd[1:]):
        assert b.mean_speed <= a.mean_speed + 0.02


@pytest.mark.gpu
def test_run_sweep_records_and_speed_factors():
    sc = fp.make_scenario("mini", fp.make_plaza(4.0, 2))
    spec = hz.SweepSpec([1, 2], [5, 10, 20], [3], steps=5, repetitions=1)
    recs = hz.run_sweep(spec, sc, 1)
    assert len(recs) == 6
    for r in recs:
        assert (r.scenario, r.v_max, r.steps) == ("mini", 3, 5)
        assert r.wall_time_s >= 0.0 and r.wall_time_s + 1e-3 >= r.plan_time_s + r.move_time_s
    rows = hz.speed_factor(recs)
    assert [r.cores for r in rows] == [1, 2] * 3
    assert hz.parse_run_csv(hz.runs_to_csv(recs))[0].agents_initial == 5


@pytest.mark.gpu
def test_realtime_capacity_on_the_device_caps_at_free_cells():
    sc = fp.make_scenario("mini", fp.make_plaza(8.0, 2))  # 20x20, 324 free cells
    r = hz.realtime_capacity_scenario(sc, 4, 1, 1, budget_steps=3, start_n=10)
    assert r.capped and r.capacity == sc.grid.free_cell_count()
