"""BASELINE configurations at full size on the GPU, through size-independent properties (the
oracle cannot follow 1e6-1e7 agents for many steps in test time; its bit-exactness is pinned on
the smaller cases): determinism, equality of the graph-replayed run() with per-call step(),
equality of the strip-decomposed plan with the full plan, and state invariants -- one agent per
cell, occupancy <-> positions, conservation of agents, walls never entered, hops <= v_max."""
import numpy as np
import pytest

from paper_0911_2900_b200 import fastped as fp
from paper_0911_2900_b200 import scenarios
from paper_0911_2900_b200.dist import strip_bounds

pytestmark = pytest.mark.gpu


def check_invariants(dev, wl, x0, y0, a0):
    x, y, a = dev.agents()
    al = a.astype(bool)
    assert not (al & ~a0.astype(bool)).any(), "a dead agent came back"
    W = wl.grid.width
    if wl.grid.boundary == fp.PERIODIC_X:
        ddx = np.abs(x - x0)
        ddx = np.minimum(ddx, W - ddx)
    else:
        ddx = np.abs(x - x0)
    hop = np.maximum(ddx, np.abs(y - y0))
    assert (hop[al] <= wl.roster.v_max[al]).all()
    assert (wl.grid.cells[y[al], x[al]] != fp.WALL).all()
    occ = dev.occupancy()
    assert (occ[y[al], x[al]] == np.flatnonzero(al)).all()
    assert (occ >= 0).sum() == al.sum() == dev.alive


@pytest.mark.timeout(900)
@pytest.mark.parametrize("config,steps", [("plaza", 40), ("ring", 40), ("room", 60)])
def test_run_is_deterministic_and_equals_stepping(config, steps):
    wl = scenarios.build(config)
    p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=steps)

    def fresh():
        st = fp.SimState(wl.grid, None, wl.roster)
        if wl.potential:
            st.set_potential(wl.potential, wl.drive_gradient)
        return st

    a, b, c = fresh(), fresh(), fresh()
    ra = fp.run(a, p)
    rb = fp.run(b, p)
    assert fp.state_hash(a) == fp.state_hash(b) and ra.exited == rb.exited
    p1 = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
    ex = disp = 0
    for _ in range(steps):
        x0, y0, a0 = c.agents()
        s = fp.step(c, p1)
        ex += s.exited
        disp += s.displacement_cells
        check_invariants(c, wl, x0, y0, a0)
    assert fp.state_hash(c) == fp.state_hash(a)
    assert ex == ra.exited and disp == ra.displacement_cells


@pytest.mark.timeout(900)
def test_plaza_strip_plan_equals_full_plan():
    wl = scenarios.build("plaza")
    p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=30)
    full = fp.SimState(wl.grid, None, wl.roster)
    fp.run(full, p)  # a crowded state
    x, y, a = full.agents()
    ro = fp.Roster(x.copy(), y.copy(), wl.roster.v_max.copy(), a.copy())
    ranks = [fp.SimState(wl.grid, full.field(), ro, step=full.step) for _ in range(2)]
    fp.plan_phase(full, p)
    fdx, fdy = full.desired()
    sdx, sdy = np.zeros_like(fdx), np.zeros_like(fdy)
    for r, st in enumerate(ranks):
        lo, hi = strip_bounds(wl.grid.width, r, 2)
        st.plan_strip(p.k_s, p.seed, lo, hi)
        dx, dy = st.desired()
        sdx += dx
        sdy += dy
    al = a.astype(bool)
    assert np.array_equal(sdx[al], fdx[al]) and np.array_equal(sdy[al], fdy[al])


@pytest.mark.timeout(1200)
def test_obstacles_config5_full_size_invariants():
    """Config 5: 40000x10000 (4e8 cells), ~15% rectangle walls, 1e7 agents, mixed v_max 2..5."""
    wl = scenarios.build("obstacles")
    dev = fp.SimState(wl.grid, None, wl.roster)
    p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
    for _ in range(3):
        x0, y0, a0 = dev.agents()
        fp.step(dev, p)
        check_invariants(dev, wl, x0, y0, a0)
