"""Parity of the CUDA path (through the C ABI) with the CPU restatement (oracle/), which is in
turn pinned to the reference (tests/test_oracle_vs_reference.py) and to the committed golden
fixtures (tests/test_golden.py).  Integer/index results must be bit-exact; fp64 fields and
weights must be bitwise equal; fp32 choice probabilities within 1e-6 relative."""
import numpy as np
import pytest

import oracle as O
from paper_0911_2900_b200 import fastped as fp
from tests.helpers import EXIT, FREE, WALL, from_rows, random_grid, random_periodic

pytestmark = pytest.mark.gpu

PROB_RTOL = 1e-6  # north star: choice probabilities within 1e-6 relative (fp32)


def pair(cells, x, y, v, boundary=0, potential=0, g=0.0, alive=None, step=0, field=None):
    """The same SimState on the device and in the oracle (device computes its own field)."""
    cells = np.ascontiguousarray(cells, np.uint8)
    n = len(x)
    v = np.broadcast_to(np.asarray(v, np.int32), (n,)).copy()
    al = np.ones(n, np.uint8) if alive is None else np.asarray(alive, np.uint8)
    grid = fp.Grid(cells, 0.4, boundary)
    dev = fp.SimState(grid, field, fp.Roster(np.asarray(x, np.int32), np.asarray(y, np.int32), v, al), step=step)
    if potential:
        dev.set_potential(potential, g)
    f = O.static_field(cells, boundary) if field is None else field
    orc = O.State(cells, f, x, y, v, alive=al, boundary=boundary, step=step, potential=potential,
                  drive_gradient=g)
    return dev, orc


def assert_same_state(dev, orc, msg=""):
    x, y, a = dev.agents()
    assert (a == orc.alive).all(), msg
    al = a.astype(bool)
    assert (x[al] == orc.x[al]).all() and (y[al] == orc.y[al]).all(), msg
    assert dev.alive == orc.alive_count, msg


# ---------------------------------------------------------------------------------- field
@pytest.mark.parametrize("boundary", [0, 1])
def test_field_bitwise_random(boundary):
    r = np.random.default_rng(71 + boundary)
    for _ in range(20):
        w, h = int(r.integers(5, 80)), int(r.integers(5, 60))
        cells = random_grid(r, w, h, 0.3 * r.random(), int(r.integers(0, 7))) if boundary == 0 \
            else random_periodic(r, w, h, 0.3 * r.random())
        if boundary:
            for _ in range(int(r.integers(0, 4))):
                cells[int(r.integers(1, h - 1)), int(r.integers(0, w))] = EXIT
        got = fp.compute_static_field(fp.Grid(cells, 0.4, boundary))
        want = O.static_field(cells, boundary)
        assert got.tobytes() == want.tobytes()


def test_field_bitwise_room_1000():
    """Config 2 geometry (1e6 cells): the device field equals the Dijkstra bit for bit."""
    from paper_0911_2900_b200 import scenarios
    wl = scenarios.room(n=10)
    got = fp.compute_static_field(wl.grid)
    want = O.static_field(wl.grid.cells, 0)
    assert got.tobytes() == want.tobytes()


def test_field_bitwise_obstacles():
    """A config-5-like obstacle field (rectangles, 15% walls, pockets)."""
    from paper_0911_2900_b200 import scenarios
    wl = scenarios.obstacles(n=10, width=1200, height=700)
    got = fp.compute_static_field(wl.grid)
    want = O.static_field(wl.grid.cells, 0)
    assert got.tobytes() == want.tobytes()


# ---------------------------------------------------------------------------------- order
@pytest.mark.parametrize("n", [0, 1, 2, 3, 5, 17, 1000, 65537, 1_000_000, 10_000_000])
def test_movement_order_matches_fisher_yates(n):
    for seed, step in ((1, 0), (99, 395)):
        got = fp.movement_order(n, seed, step)
        want = O.movement_order(n, seed, step)
        assert (got == want).all()


# ---------------------------------------------------------------------------------- plan
def _random_state(r, boundary=0, mixed=True, dead_frac=0.0):
    if boundary == 0:
        cells = random_grid(r, int(r.integers(15, 90)), int(r.integers(15, 90)), 0.05 + 0.2 * r.random(),
                            1 + int(r.integers(8)))
    else:
        cells = random_periodic(r, int(r.integers(12, 90)), int(r.integers(8, 40)), 0.1 * r.random())
    nfree = int((cells == FREE).sum())
    n = max(1, min(1000, nfree // 3))
    x, y = O.spawn_agents(cells, n, int(r.integers(1, 1 << 31)))
    v = (1 + r.integers(0, 5, n)).astype(np.int32) if mixed else np.full(n, 1 + int(r.integers(5)), np.int32)
    alive = (r.random(n) >= dead_frac).astype(np.uint8)
    return cells, x, y, v, alive


@pytest.mark.parametrize("case", range(12))
def test_plan_desired_bitwise(case):
    r = np.random.default_rng(5000 + case)
    boundary = 1 if case % 4 == 3 else 0
    potential = 1 if case in (3, 11) else 0
    cells, x, y, v, alive = _random_state(r, boundary, mixed=case % 2 == 0, dead_frac=0.1 if case % 3 == 0 else 0)
    dev, orc = pair(cells, x, y, v, boundary, potential, 1.0 if case == 3 else 8.0, alive=alive,
                    step=int(r.integers(0, 400)))
    for k_s, seed in ((1.2, 1), (0.0, 404), (3.0, 2**63 + 5)):
        fp.plan_phase(dev, fp.SimParams(k_s=k_s, seed=seed))
        orc.plan(k_s, seed)
        dx, dy = dev.desired()
        al = alive.astype(bool)
        assert (dx[al] == orc.dx[al]).all() and (dy[al] == orc.dy[al]).all(), (k_s, seed)


def test_plan_skips_dead_and_empty():  # tests/test_engine.cpp:76-94
    cells = from_rows(["#####", "#...#", "#..E#", "#####"])
    dev, orc = pair(cells, np.array([1, 2], np.int32), np.array([1, 1], np.int32), 1, alive=[1, 0])
    dev.set_desired(np.array([1, -7], np.int32), np.array([1, -7], np.int32))
    fp.plan_phase(dev, fp.SimParams(), fp.ScheduleParams(4))
    dx, dy = dev.desired()
    assert (dx[1], dy[1]) == (-7, -7)
    empty = fp.SimState(fp.from_rows(["###", "#E#", "###"]), None, fp.roster([], 1))
    fp.plan_phase(empty, fp.SimParams(), fp.ScheduleParams(4))
    s = fp.step(empty, fp.SimParams(), fp.ScheduleParams(2))
    assert (s.alive, s.exited, s.displacement_cells) == (0, 0, 0)


def test_choice_weights_and_probabilities():
    r = np.random.default_rng(77)
    cells, x, y, v, _ = _random_state(r, 0, mixed=True)
    dev, orc = pair(cells, x, y, v)
    for i in range(0, len(x), max(1, len(x) // 50)):
        cx, cy, w, p = dev.choice(i, 1.2)
        wo, cxo, cyo = orc.weights(i, 1.2)
        assert (cx == cxo).all() and (cy == cyo).all()
        assert w.tobytes() == wo.tobytes()
        pref = wo / wo.sum()
        nz = pref > 0
        assert np.all(np.abs(p[nz] - pref[nz]) <= PROB_RTOL * pref[nz] + 1e-30)
        assert (p[~nz] == 0).all()


def test_narrow_periodic_corridor():  # tests/test_planning.cpp:114-123 through the device
    cells = from_rows(["######", "......", "......", "......", "######"])
    dev, orc = pair(cells, np.array([2], np.int32), np.array([2], np.int32), 4, boundary=1)
    cx, cy, w, p = dev.choice(0, 1.2)
    assert list(zip(cx, cy)) == orc.candidates(0) and len(cx) == 18


# ---------------------------------------------------------------------------------- motion
def test_motion_micro_cases():  # tests/test_engine.cpp:96-158
    g = from_rows(["#####", "#...#", "#####"])
    dev, _ = pair(g, np.array([2], np.int32), np.array([1], np.int32), 4)
    dev.set_desired(np.array([2], np.int32), np.array([1], np.int32))
    mv = fp.move_phase(dev, fp.SimParams())
    assert dev.agents()[0][0] == 2 and mv.displacement_cells == 0 and mv.exited == []

    g = from_rows(["#######", "#.....#", "#######"])
    dev, orc = pair(g, np.array([1, 4], np.int32), np.array([1, 1], np.int32), 4)
    dev.set_desired(np.array([5, 4], np.int32), np.array([1, 1], np.int32))
    fp.move_phase(dev, fp.SimParams())
    x, y, a = dev.agents()
    assert (x[0], x[1]) == (3, 4)

    g = from_rows(["#####", "#..E#", "#####"])
    dev, _ = pair(g, np.array([1], np.int32), np.array([1], np.int32), 2)
    dev.set_desired(np.array([3], np.int32), np.array([1], np.int32))
    mv = fp.move_phase(dev, fp.SimParams())
    assert mv.exited == [0] and dev.alive == 0 and mv.displacement_cells == 2
    assert (dev.occupancy() == -1).all()


@pytest.mark.parametrize("case", range(10))
def test_motion_injected_desired_bitwise(case):
    """Random desired cells (inside and beyond the ball, through walls and exits)."""
    r = np.random.default_rng(900 + case)
    boundary = 1 if case % 5 == 4 else 0
    cells, x, y, v, alive = _random_state(r, boundary, mixed=True, dead_frac=0.05)
    dev, orc = pair(cells, x, y, v, boundary, alive=alive)
    n = len(x)
    h, w = cells.shape
    dx = (x + r.integers(-6, 7, n)).astype(np.int32)
    dy = np.clip(y + r.integers(-6, 7, n), 0, h - 1).astype(np.int32)
    if boundary == 0:
        dx = np.clip(dx, 0, w - 1).astype(np.int32)
    dev.set_desired(dx, dy)
    orc.dx[:] = dx
    orc.dy[:] = dy
    for s in range(3):
        seed = int(r.integers(1, 1 << 40))
        mv = fp.move_phase(dev, fp.SimParams(seed=seed))
        ex, disp = orc.move(seed)
        assert mv.exited == ex.tolist() and mv.displacement_cells == disp
        assert_same_state(dev, orc, f"round {s}")
        assert (dev.occupancy().ravel() == orc.occ).all()


@pytest.mark.parametrize("case", range(20))
def test_trajectories_bitwise(case):
    """tests/acceptance.cpp:114-143 shape: 20 scenarios, 50 steps, positions + alive + exit
    order every step, and the state hash."""
    r = np.random.default_rng(0xACCE55 + 17 * case)
    boundary = 1 if case % 5 == 2 else 0
    potential = 1 if case % 10 == 2 else 0
    cells, x, y, v, _ = _random_state(r, boundary, mixed=case % 3 == 0)
    dev, orc = pair(cells, x, y, v, boundary, potential, 8.0)
    params = fp.SimParams(seed=int(r.integers(1, 1 << 62)))
    for s in range(50):
        fp.plan_phase(dev, params)
        mv = fp.move_phase(dev, params)
        dev.step = dev.step + 1
        ex, disp = orc.step_once(params.k_s, params.seed)
        assert mv.exited == ex.tolist(), f"step {s}"
        assert mv.displacement_cells == disp
        assert_same_state(dev, orc, f"step {s}")
        assert fp.state_hash(dev) == orc.hash()


def test_run_matches_stepping():
    r = np.random.default_rng(31)
    cells, x, y, v, _ = _random_state(r, 0, mixed=False)
    dev, orc = pair(cells, x, y, v)
    rs = fp.run(dev, fp.SimParams(seed=8080, steps=40))
    for _ in range(40):
        orc.step_once(1.2, 8080)
    assert rs.steps == 40 and dev.step == 40
    assert_same_state(dev, orc)
    assert fp.state_hash(dev) == orc.hash()
    assert rs.plan_time_s + rs.move_time_s <= rs.wall_time_s + 1e-3


@pytest.mark.parametrize("wide", [False, True])
def test_potential_change_between_graph_steps(wide):
    """state.hpp: potential / drive_gradient are mutable fields of SimState.  step() and run()
    replay captured graphs that hold the plan kernel's parameters by value, so a change of the
    gradient (DriveX -> DriveX) or of the potential kind between steps must re-capture them:
    the trajectory follows the oracle stepped with the same changes.  The narrow ring plans
    through the untiled variant, the wide one through the tiled weight plane."""
    r = np.random.default_rng(0x9AD1 + wide)
    cells = random_periodic(r, 300 if wide else 40, 24, 0.04)
    for _ in range(3):
        cells[int(r.integers(1, 23)), int(r.integers(0, cells.shape[1]))] = EXIT
    nfree = int((cells == FREE).sum())
    x, y = O.spawn_agents(cells, nfree // 4, 77)
    dev, orc = pair(cells, x, y, 3, 1, 1, 8.0)
    p = fp.SimParams(k_s=1.2, seed=4242)
    schedule = [(1, 8.0), (1, 2.5), (1, -6.0), (0, 0.0), (1, 11.0)]
    for i, (kind, g) in enumerate(schedule):
        dev.set_potential(kind, g)
        orc.s.potential, orc.s.drive_gradient = kind, g
        if i % 2 == 0:
            for s in range(3):
                fp.step(dev, p)
                orc.step_once(p.k_s, p.seed)
                assert fp.state_hash(dev) == orc.hash(), f"phase {i} step {s}"
        else:
            fp.run(dev, fp.SimParams(k_s=1.2, seed=4242, steps=3))
            for s in range(3):
                orc.step_once(p.k_s, p.seed)
            assert fp.state_hash(dev) == orc.hash(), f"phase {i} run"
        assert_same_state(dev, orc, f"phase {i}")


@pytest.mark.parametrize("name", ["corridor", "ring"])
def test_config_trajectories(name):
    """Configs 1 and 3 at full size (config 3: 182,000 agents, DriveX on the ring)."""
    from paper_0911_2900_b200 import scenarios
    wl = scenarios.build(name)
    ro = wl.roster
    steps = 396 if name == "corridor" else 8
    dev, orc = pair(wl.grid.cells, ro.x, ro.y, ro.v_max, wl.grid.boundary, wl.potential, wl.drive_gradient)
    for s in range(steps):
        fp.step(dev, fp.SimParams(k_s=wl.k_s, seed=wl.seed))
        orc.step_once(wl.k_s, wl.seed)
        if s % 20 == 0 or s == steps - 1:
            assert_same_state(dev, orc, f"{name} step {s}")
    assert fp.state_hash(dev) == orc.hash()


def test_config2_room_steps():
    from paper_0911_2900_b200 import scenarios
    for v in (1, 4, 5):
        wl = scenarios.room(v=v)
        ro = wl.roster
        dev, orc = pair(wl.grid.cells, ro.x, ro.y, ro.v_max)
        for s in range(12):
            fp.step(dev, fp.SimParams(seed=wl.seed))
            orc.step_once(1.2, wl.seed)
        assert_same_state(dev, orc, f"v={v}")
        assert fp.state_hash(dev) == orc.hash()


def test_plan_repeatable_under_load():
    """Race detector for the tiled plan kernel's slot pipeline: the dense ring (many tiles per
    CTA, > 512 agents in a tile) planned repeatedly must give identical desired cells, equal to
    the oracle's."""
    from paper_0911_2900_b200 import scenarios
    wl = scenarios.ring()
    ro = wl.roster
    dev, orc = pair(wl.grid.cells, ro.x, ro.y, ro.v_max, wl.grid.boundary, wl.potential, wl.drive_gradient)
    orc.plan(wl.k_s, wl.seed)
    for _ in range(8):
        fp.plan_phase(dev, fp.SimParams(k_s=wl.k_s, seed=wl.seed))
        dx, dy = dev.desired()
        assert (dx == orc.dx).all() and (dy == orc.dy).all()


def test_plaza_sampled_plan_and_invariants():
    """Config 4 at full size (1e8 cells, 1e6 agents): planned cells of a sample of agents equal
    the oracle's choose_desired_cell; after motion the state is consistent (occupancy <-> positions),
    conservation holds and nobody moved farther than v_max."""
    import ctypes as C
    from paper_0911_2900_b200 import scenarios
    wl = scenarios.plaza()
    ro = wl.roster
    dev = fp.SimState(wl.grid, None, ro)
    field = dev.field()
    fp.plan_phase(dev, fp.SimParams(seed=wl.seed))
    dx, dy = dev.desired()
    # oracle on a sample: build a small oracle state view over the full grid
    orc = O.State(wl.grid.cells, field, ro.x, ro.y, ro.v_max)
    rng = np.random.default_rng(5)
    for i in rng.choice(len(ro.x), 2000, replace=False):
        ox, oy = C.c_int32(), C.c_int32()
        O.lib().orc_choose_desired.argtypes = [C.POINTER(O.OrcState), C.c_int32, C.c_double, C.c_uint64,
                                               C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        O.lib().orc_choose_desired(C.byref(orc.s), int(i), 1.2, wl.seed, C.byref(ox), C.byref(oy))
        assert (dx[i], dy[i]) == (ox.value, oy.value), i
    x0, y0, _ = dev.agents()
    mv = fp.move_phase(dev, fp.SimParams(seed=wl.seed))
    x1, y1, a1 = dev.agents()
    al = a1.astype(bool)
    assert np.maximum(np.abs(x1 - x0), np.abs(y1 - y0))[al].max() <= 4
    assert dev.alive + len(mv.exited) == len(ro.x)
    occ = dev.occupancy()
    assert (occ[y1[al], x1[al]] == np.nonzero(al)[0]).all()
    assert (occ >= 0).sum() == al.sum()


def _pocket_grid(r, w=120, h=90):
    """Closed rooms with exits, plus walled pockets (enclosed free cells: unreachable, S = inf)
    scattered through them; thin (1-cell) pocket walls so reachable agents see pocket cells inside
    their balls."""
    c = random_grid(r, w, h, 0.05, 3)
    for _ in range(25):
        pw, ph = int(r.integers(2, 7)), int(r.integers(2, 7))
        x0, y0 = int(r.integers(2, w - pw - 3)), int(r.integers(2, h - ph - 3))
        c[y0 - 1:y0 + ph + 1, x0 - 1:x0 + pw + 1] = WALL
        c[y0:y0 + ph, x0:x0 + pw] = FREE
    return c


@pytest.mark.parametrize("case", range(4))
def test_plan_flagged_centres(case):
    """The weight plane's exact-path flag (plane.cu): agents inside unreachable pockets (all
    weights 1), agents with pocket cells within Chebyshev 5 (zero-weight candidates), and steep
    fields (k_s = 8: weights spanning > 2^60 in a ball) -- every decision equal to the oracle's."""
    r = np.random.default_rng(7100 + case)
    cells = _pocket_grid(r)
    free = np.argwhere(cells == FREE)
    pick = r.choice(len(free), size=min(1500, len(free) // 3), replace=False)
    y, x = free[pick, 0].astype(np.int32), free[pick, 1].astype(np.int32)
    v = r.integers(1, 6, len(x)).astype(np.int32) if case % 2 else np.full(len(x), 5, np.int32)
    dev, orc = pair(cells, x, y, v, step=int(r.integers(0, 300)))
    f = O.static_field(cells, 0)
    assert np.isinf(f[y, x]).any(), "no agent inside a pocket"
    for k_s, seed in ((1.2, 3), (8.0, 77), (20.0, 5)):
        fp.plan_phase(dev, fp.SimParams(k_s=k_s, seed=seed))
        orc.plan(k_s, seed)
        dx, dy = dev.desired()
        assert (dx == orc.dx).all() and (dy == orc.dy).all(), (k_s, seed)
