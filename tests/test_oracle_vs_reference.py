"""Pins the C restatement against the UNMODIFIED reference compiled here (oracle/_ref):
bitwise field, candidates, weights, desired cells, trajectories, exit order and state hash.
Skipped where oracle/_ref was not built (the reference is absent on the GPU box)."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import FREE, random_grid, random_periodic

pytestmark = pytest.mark.skipif(not O.have_reference(), reason="oracle/_ref not built")


def test_rng_and_blocksize_match():
    r = np.random.default_rng(1)
    for _ in range(2000):
        s, a, t, d = (int(v) for v in r.integers(0, 2**63, 4, dtype=np.int64))
        assert O.rng_u64(s, a, t, d) == O.ref().ref_rng_u64(s, a, t, d)
    for n, c in [(0, 1), (5, 3), (100000, 8), (10**7, 7), (3, 8)]:
        assert O.compute_blocksize(n, c) == O.ref().ref_compute_blocksize(n, c)


@pytest.mark.parametrize("boundary", [0, 1])
def test_field_bitwise(boundary):
    r = np.random.default_rng(555 + boundary)
    for _ in range(15):
        w, h = int(r.integers(8, 60)), int(r.integers(5, 40))
        cells = random_grid(r, w, h, r.random() * 0.3, int(r.integers(0, 6))) if boundary == 0 \
            else random_periodic(r, w, h, r.random() * 0.3)
        if boundary == 1:
            k = int(r.integers(0, 4))
            for _ in range(k):
                cells[int(r.integers(1, h - 1)), int(r.integers(0, w))] = 2
        a = O.static_field(cells, boundary)
        b = O.ref_static_field(cells, boundary)
        assert a.tobytes() == b.tobytes()


def _scenario(r, boundary, mixed_v=False):
    w, h = int(r.integers(12, 50)), int(r.integers(12, 40))
    if boundary == 0:
        cells = random_grid(r, w, h, 0.05 + 0.2 * r.random(), 1 + int(r.integers(6)))
    else:
        cells = random_periodic(r, max(w, 12), h, 0.1 * r.random())
    nfree = int((cells == FREE).sum())
    n = max(1, min(300, nfree // 3))
    x, y = O.spawn_agents(cells, n, int(r.integers(1, 1 << 30)))
    v = (1 + r.integers(0, 5, n)).astype(np.int32) if mixed_v else np.full(n, 1 + int(r.integers(5)), np.int32)
    return cells, x, y, v


@pytest.mark.parametrize("case", range(6))
def test_candidates_and_weights_bitwise(case):
    r = np.random.default_rng(100 + case)
    boundary = case % 2
    cells, x, y, v = _scenario(r, boundary, mixed_v=True)
    f = O.static_field(cells, boundary)
    pot = 1 if (boundary == 1 and case % 3 == 0) else 0
    a = O.State(cells, f, x, y, v, boundary=boundary, potential=pot, drive_gradient=1.0)
    b = O.RefState(cells, f, x, y, v, boundary=boundary, potential=pot, drive_gradient=1.0)
    for i in range(len(x)):
        wa, xa, ya = a.weights(i, 1.2)
        wb, xb, yb = b.weights(i, 1.2)
        assert (xa == xb).all() and (ya == yb).all()
        assert wa.tobytes() == wb.tobytes()


@pytest.mark.parametrize("case", range(8))
def test_trajectories_bitwise(case):
    """plan + move for 25 steps: positions, alive, exit order and hash every step."""
    r = np.random.default_rng(0xACCE55 + case)
    boundary = 1 if case in (3, 7) else 0
    cells, x, y, v = _scenario(r, boundary, mixed_v=(case % 4 == 1))
    f = O.static_field(cells, boundary)
    pot = 1 if case == 7 else 0
    seed = int(r.integers(1, 1 << 40))
    a = O.State(cells, f, x, y, v, boundary=boundary, potential=pot, drive_gradient=8.0)
    b = O.RefState(cells, f, x, y, v, boundary=boundary, potential=pot, drive_gradient=8.0)
    for s in range(25):
        ea, da = a.step_once(1.2, seed)
        eb, db = b.step_once(1.2, seed, cores=1 + s % 4)
        xb, yb, alb = b.agents()
        assert (a.x == xb).all() and (a.y == yb).all() and (a.alive == alb).all(), f"step {s}"
        assert ea.tolist() == eb.tolist() and da == db
        assert a.hash() == b.hash()
        assert (a.occ.reshape(a.h, a.w) == b.occupancy()).all()


def test_spawn_matches():
    r = np.random.default_rng(4)
    cells = random_grid(r, 40, 30, 0.2, 2)
    for seed in (1, 2, 99):
        xa, ya = O.spawn_agents(cells, 200, seed)
        xb = np.empty(200, np.int32)
        yb = np.empty(200, np.int32)
        assert O.ref().ref_spawn_agents(40, 30, cells.ravel(), 0, 200, 4, seed, xb, yb) == 0
        assert (xa == xb).all() and (ya == yb).all()


def test_exp_is_the_references():
    r = np.random.default_rng(9)
    for xv in r.uniform(-20, 20, 5000):
        assert O.lib().orc_exp(xv) == O.ref().ref_exp(xv)
