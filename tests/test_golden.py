"""Golden fixtures produced by running the reference itself (oracle/_ref, the unmodified headers;
tests/golden/make_golden.py) on five seeded scenarios.  They pin the C restatement (CPU tests)
and the CUDA engine through the C ABI (GPU tests) without /root/reference at test time:
static field bitwise, and per step the desired cells, movement order, positions, alive flags,
exit ids in processing order, displacement and state_hash -- all bit-exact."""
import glob
import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(HERE, "*.npz"))
               if not os.path.basename(p).startswith("full_"))  # full_*: tests/test_fullsize_golden.py


def load(name):
    return dict(np.load(os.path.join(HERE, name + ".npz")))


def per_step(flat, off, s):
    return flat[off[s]:off[s + 1]]


def test_fixtures_present():
    assert len(CASES) >= 5, "run tests/golden/make_golden.py"


@pytest.mark.parametrize("name", CASES)
def test_restatement_reproduces_reference_fixture(name):
    g = load(name)
    field = O.static_field(g["cells"], int(g["boundary"]))
    assert np.array_equal(field.view(np.uint64), g["field"].view(np.uint64))
    st = O.State(g["cells"], field, g["x0"], g["y0"], g["v_max"], boundary=int(g["boundary"]),
                 potential=int(g["potential"]), drive_gradient=float(g["drive_gradient"]))
    k_s, seed = float(g["k_s"]), int(g["seed"])
    for s in range(len(g["pos"])):
        alive_ids = np.flatnonzero(st.alive)
        perm = O.movement_order(len(alive_ids), seed, s)
        assert np.array_equal(alive_ids[perm] if len(alive_ids) else alive_ids,
                              per_step(g["order"], g["order_off"], s)), (name, s)
        st.plan(k_s, seed)
        al = st.alive.astype(bool)
        assert np.array_equal(st.dx[al], g["desired"][s][0][al]), (name, s)
        assert np.array_equal(st.dy[al], g["desired"][s][1][al]), (name, s)
        ex, disp = st.move(seed)
        st.step = st.step + 1
        assert np.array_equal(np.asarray(ex, np.int64), per_step(g["exited"], g["exited_off"], s)), (name, s)
        assert disp == g["displacement"][s], (name, s)
        assert np.array_equal(st.alive, g["alive"][s]), (name, s)
        al = st.alive.astype(bool)
        assert np.array_equal(st.x[al], g["pos"][s][0][al]) and np.array_equal(st.y[al], g["pos"][s][1][al])
        assert st.hash() == int(g["state_hash"][s]), (name, s)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_cuda_engine_reproduces_reference_fixture(name):
    from paper_0911_2900_b200 import fastped as fp
    g = load(name)
    grid = fp.Grid(g["cells"], 0.4, int(g["boundary"]))
    ro = fp.Roster(g["x0"].copy(), g["y0"].copy(), g["v_max"].copy(), np.ones(len(g["x0"]), np.uint8))
    dev = fp.SimState(grid, None, ro)  # the device computes its own static field
    assert np.array_equal(dev.field().ravel().view(np.uint64), g["field"].ravel().view(np.uint64))
    if int(g["potential"]):
        dev.set_potential(int(g["potential"]), float(g["drive_gradient"]))
    p = fp.SimParams(k_s=float(g["k_s"]), seed=int(g["seed"]), steps=1)
    for s in range(len(g["pos"])):
        al0 = dev.agents()[2].astype(bool)
        fp.plan_phase(dev, p)
        dx, dy = dev.desired()
        assert np.array_equal(dx[al0], g["desired"][s][0][al0]), (name, s)
        assert np.array_equal(dy[al0], g["desired"][s][1][al0]), (name, s)
        out = fp.move_phase(dev, p)
        assert np.array_equal(dev.last_order(), per_step(g["order"], g["order_off"], s)), (name, s)
        dev.step = dev.step + 1
        assert np.array_equal(np.asarray(out.exited, np.int64), per_step(g["exited"], g["exited_off"], s)), (name, s)
        assert out.displacement_cells == g["displacement"][s], (name, s)
        x, y, a = dev.agents()
        assert np.array_equal(a, g["alive"][s]), (name, s)
        al = a.astype(bool)
        assert np.array_equal(x[al], g["pos"][s][0][al]) and np.array_equal(y[al], g["pos"][s][1][al]), (name, s)
        assert fp.state_hash(dev) == int(g["state_hash"][s]), (name, s)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_cuda_run_reaches_reference_final_state(name):
    """The device-resident run() loop (CUDA graphs) over all fixture steps."""
    from paper_0911_2900_b200 import fastped as fp
    g = load(name)
    grid = fp.Grid(g["cells"], 0.4, int(g["boundary"]))
    ro = fp.Roster(g["x0"].copy(), g["y0"].copy(), g["v_max"].copy(), np.ones(len(g["x0"]), np.uint8))
    dev = fp.SimState(grid, g["field"], ro)
    if int(g["potential"]):
        dev.set_potential(int(g["potential"]), float(g["drive_gradient"]))
    steps = len(g["pos"])
    r = fp.run(dev, fp.SimParams(k_s=float(g["k_s"]), seed=int(g["seed"]), steps=steps))
    assert r.exited == len(g["exited"])
    assert r.displacement_cells == int(g["displacement"].sum())
    assert fp.state_hash(dev) == int(g["state_hash"][-1])
