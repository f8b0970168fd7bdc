"""BASELINE configurations at full size on the GPU, through size-independent properties (the
oracle cannot follow 1e6-1e7 agents for many steps in test time; its bit-exactness is pinned on
the smaller cases): determinism, equality of the graph-replayed run() with per-call step(),
equality of the strip-decomposed plan with the full plan, and state invariants -- one agent per
cell, occupancy <-> positions, conservation of agents, walls never entered, hops <= v_max."""
import numpy as np
import pytest

from paper_0911_2900_b200 import fastped as fp
from paper_0911_2900_b200 import scenarios

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
