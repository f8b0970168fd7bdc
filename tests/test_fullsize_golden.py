"""Full-size trajectory parity: BASELINE.json's configurations at their full sizes and lengths,
stepped through the C ABI on the GPU and compared EVERY STEP against fixtures the reference
engine itself produced (tests/golden/make_fullsize.py over oracle/_ref):

    state_hash after the step (state.hpp:80-95), alive count, displacement, exited ids in
    processing order (engine.hpp:123-128), and a digest of the desired cells (plan_phase).

This is the reference's trajectory contract (tests/acceptance.cpp:114-143) at the bench's own
scale, including the jammed exit-queue regime late in the plaza and room runs.  The run() path
(CUDA graphs, one host sync) is checked against the same fixture's totals and final hash.
The workloads are rebuilt from the product's generators (paper_0911_2900_b200/scenarios.py);
the fixture's sha256 of the cells and the roster pins that they are the reference's inputs.
"""
import ctypes as C
import os

import numpy as np
import pytest

import oracle.configs as OC
from paper_0911_2900_b200 import fastped as fp
from paper_0911_2900_b200 import scenarios

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ["corridor", "room_v1", "room_v2", "room_v3", "room_v4", "room_v5", "ring", "plaza", "obstacles"]


def fixture(name):
    path = os.path.join(GOLD, f"full_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    return np.load(path, allow_pickle=False)


def workload(f):
    kw = eval(str(f["kwargs"]), {})  # a dict literal written by make_fullsize.py
    wl = scenarios.build(str(f["config"]), **kw)
    assert OC.cells_digest(wl.grid.cells) == str(f["cells_sha256"]), "geometry differs from the fixture's"
    assert OC.roster_digest(wl.roster.x, wl.roster.y, wl.roster.v_max) == str(f["roster_sha256"]), \
        "roster differs from the reference's spawn"
    return wl


def fresh(wl):
    st = fp.SimState(wl.grid, None, wl.roster)
    if wl.potential:
        st.set_potential(wl.potential, wl.drive_gradient)
    return st


def exited_ids(st, n):
    buf = np.empty(max(n, 1), np.uint32)
    k = C.c_uint32()
    fp._check(fp.library().fp_get_exited(st._ctx, buf, len(buf), C.byref(k)), st._ctx)
    return buf[: k.value]


@pytest.mark.parametrize("name", NAMES)
def test_fixture_roster_is_the_configs_roster(name):
    """CPU: the checker-side generators (oracle/configs.py) reproduce the fixture's inputs
    (plaza / obstacles rosters are checked on the GPU box, where building them is cheap)."""
    f = fixture(name)
    if str(f["config"]) in ("plaza", "obstacles"):
        pytest.skip("built in the GPU test")
    cfg = OC.build(str(f["config"]), **eval(str(f["kwargs"]), {}))
    assert OC.cells_digest(cfg.cells) == str(f["cells_sha256"])
    assert OC.roster_digest(cfg.x, cfg.y, cfg.v) == str(f["roster_sha256"])
    assert len(f["state_hash"]) == int(f["steps"]) and f["exited_off"][-1] == len(f["exited"])


def test_restatement_follows_full_corridor():
    """CPU: the C restatement (oracle/oracle.c) reproduces the reference's full-length config-1
    trajectory fixture step by step (the larger fixtures take the oracle minutes)."""
    import oracle as O
    f = fixture("corridor")
    cfg = OC.build("corridor")
    st = O.State(cfg.cells, O.static_field(cfg.cells, 0), cfg.x, cfg.y, cfg.v)
    off = f["exited_off"]
    for s in range(int(f["steps"])):
        ex, disp = st.step_once(cfg.k_s, cfg.seed)
        assert ex.tolist() == f["exited"][off[s]:off[s + 1]].tolist() and disp == int(f["displacement"][s])
        assert st.hash() == int(f["state_hash"][s])


@pytest.mark.gpu
@pytest.mark.timeout(1800)
@pytest.mark.parametrize("name", NAMES)
def test_every_step_matches_reference(name):
    f = fixture(name)
    wl = workload(f)
    st = fresh(wl)
    assert fp.state_hash(st) == int(f["hash0"])
    p = fp.SimParams(k_s=float(f["k_s"]), seed=int(f["seed"]), steps=1)
    off = f["exited_off"]
    alive_before = wl.roster.alive.astype(bool)
    for s in range(int(f["steps"])):
        stats = fp.step(st, p)
        dx, dy = st.desired()
        assert OC.desired_digest(dx, dy, alive_before) == int(f["desired_digest"][s]), f"plan differs at step {s}"
        ex = exited_ids(st, stats.exited)
        assert ex.tolist() == f["exited"][off[s]:off[s + 1]].tolist(), f"exit order differs at step {s}"
        assert stats.alive == int(f["alive"][s]), f"alive differs at step {s}"
        assert stats.displacement_cells == int(f["displacement"][s]), f"displacement differs at step {s}"
        assert fp.state_hash(st) == int(f["state_hash"][s]), f"state differs at step {s}"
        alive_before = st.agents()[2].astype(bool)


@pytest.mark.gpu
@pytest.mark.timeout(1800)
@pytest.mark.parametrize("name", ["room_v4", "ring", "plaza", "obstacles"])
def test_run_matches_reference(name):
    """run() (graph replays, device-resident loop) over the whole fixture."""
    f = fixture(name)
    wl = workload(f)
    st = fresh(wl)
    steps = int(f["steps"])
    r = fp.run(st, fp.SimParams(k_s=float(f["k_s"]), seed=int(f["seed"]), steps=steps))
    assert r.exited == int(f["exited_off"][-1])
    assert r.displacement_cells == int(f["displacement"].sum())
    assert r.alive == int(f["alive"][-1])
    assert fp.state_hash(st) == int(f["state_hash"][-1])


@pytest.mark.gpu
@pytest.mark.timeout(1800)
@pytest.mark.parametrize("name", ["room_v5", "plaza", "obstacles"])
def test_repeated_runs_are_identical(name):
    """Race probe for the lock-free motion and plan pipelines: the same run repeated on fresh
    contexts always ends on the reference's final state (a lost occupancy update or a stale ring
    slot would show up as a divergent run, as a rare one did before the start-cell fence)."""
    f = fixture(name)
    wl = workload(f)
    steps = int(f["steps"])
    for rep in range(4):
        st = fresh(wl)
        fp.run(st, fp.SimParams(k_s=float(f["k_s"]), seed=int(f["seed"]), steps=steps))
        assert fp.state_hash(st) == int(f["state_hash"][-1]), f"repetition {rep} diverged"
