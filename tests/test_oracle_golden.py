"""Pins the C restatement (oracle/) against the reference's own golden vectors and fixtures
(SURVEY 8c), with independent brute-force checks where the reference uses them.  CPU only."""
import math

import numpy as np
import pytest

import oracle as O
from tests.helpers import EXIT, FREE, WALL, from_rows, random_grid


def state(rows, agents, v, boundary=0, field=None, potential=0, g=0.0):
    cells = from_rows(rows)
    f = O.static_field(cells, boundary) if field is None else field
    x = [a[0] for a in agents]
    y = [a[1] for a in agents]
    return O.State(cells, f, np.array(x, np.int32), np.array(y, np.int32), v, boundary=boundary,
                   potential=potential, drive_gradient=g)


def test_rng_golden_values():  # tests/test_rng.cpp:17-19
    assert O.rng_u64(0, 0, 0, 0) == 0
    assert O.rng_u64(1, 2, 3, 4) == 0xB50D425263A7BF8E
    assert O.rng_u64(42, 7, 396, 1) == 0x0374D07BEE8DB840


def test_rng_adjacent_draws_differ():  # tests/test_rng.cpp:22-28 (sampled)
    r = np.random.default_rng(12345)
    for _ in range(20000):
        s, a, t, d = (int(v) for v in r.integers(0, 2**63, 4, dtype=np.int64))
        assert O.rng_u64(s, a, t, d) != O.rng_u64(s, a, t, d + 1)


def test_unit_interval_range():  # tests/test_rng.cpp:30-40
    assert O.unit_interval(0) == 0.0
    assert O.unit_interval(2**64 - 1) < 1.0
    assert O.unit_interval(2**64 - 1) > 0.9999999999


def test_blocksize_vectors():  # tests/test_engine.cpp:35-43, tests/acceptance.cpp:97
    for n, c, want in [(100000, 8, 12500), (500000, 2, 32767), (3, 8, 1), (0, 4, 1), (32767 * 4, 4, 32767)]:
        assert O.compute_blocksize(n, c) == want
    assert O.compute_blocksize(100, 0) == -1
    assert O.compute_blocksize(-1, 2) == -1


def test_sample_index_strictness():  # tests/test_planning.cpp:133-139
    w = [1.0, 1.0]
    assert O.sample_index(w, 0.499999) == 0
    assert O.sample_index(w, 0.5) == 1
    assert O.sample_index(w, 0.0) == 0
    assert O.sample_index(w, 0.999999) == 1


def test_sample_index_scale_invariance():  # tests/test_planning.cpp:141-155
    r = np.random.default_rng(21)
    for _ in range(500):
        w = r.random(1 + r.integers(12)) + 1e-3
        u = r.random()
        base = O.sample_index(w, u)
        for k in (0.25, 0.5, 2.0, 1024.0, 3.7, 0.013):
            assert O.sample_index(w * k, u) == base


OPEN7 = ["#######", "#.....#", "#.....#", "#..E..#", "#.....#", "#.....#", "#######"]


def test_candidates_3x3_block():  # tests/test_planning.cpp:58-69
    st = state(OPEN7, [(2, 2)], 1)
    c = st.candidates(0)
    assert len(c) == 9
    assert c == sorted(c, key=lambda p: (p[1], p[0]))
    assert c[0] == (1, 1) and c[4] == (2, 2) and c[8] == (3, 3)


def test_candidates_walled_in():  # tests/test_planning.cpp:71-77
    st = state(["###", "#.#", "###"], [(1, 1)], 5)
    assert st.candidates(0) == [(1, 1)]


def test_candidates_exclude_occupied():  # tests/test_planning.cpp:79-85
    st = state(["#####", "#...#", "#...#", "#..E#", "#####"], [(1, 1), (2, 1)], 1)
    c = st.candidates(0)
    assert (1, 1) in c and (2, 1) not in c


def brute_candidates(st, i):
    """Whole-grid filter then row-major sort (the shape of tests/test_support.hpp:75-91)."""
    out = []
    px = st.x[i] % st.w if st.s.boundary else st.x[i]
    py = st.y[i]
    v = st.v_max[i]
    occ = st.occ.reshape(st.h, st.w)
    tx = np.empty(64, np.int32)
    ty = np.empty(64, np.int32)
    for y in range(st.h):
        for x in range(st.w):
            dx = x - px
            if st.s.boundary:
                alt = dx - st.w if dx > 0 else dx + st.w
                if abs(alt) < abs(dx):
                    dx = alt
            if max(abs(dx), abs(y - py)) > v:
                continue
            if st.cells[y, x] == WALL:
                continue
            if occ[y, x] not in (-1, i):
                continue
            n = O.lib().orc_trace(st.w, st.s.boundary, int(px), int(py), x, y, tx, ty, 64)
            if any(st.cells[ty[k], tx[k]] == WALL for k in range(n)):
                continue
            out.append((x, y))
    return sorted(out, key=lambda p: (p[1], p[0]))


def test_candidates_wall_segment_fixture():  # tests/test_planning.cpp:87-95
    rows = ["############", "#..........#", "#..######..#", "#..........#", "#.....E....#",
            "#..........#", "#..........#", "############"]
    st = state(rows, [(5, 4)], 4)
    assert st.candidates(0) == brute_candidates(st, 0)


def test_candidates_random_crowded_grids():  # tests/test_planning.cpp:97-112 (own seed stream)
    r = np.random.default_rng(808)
    for _ in range(25):
        v = 1 + int(r.integers(5))
        cells = random_grid(r, 14 + int(r.integers(8)), 14 + int(r.integers(8)), 0.22, 2)
        free = np.argwhere(cells == FREE)
        if len(free) < 6:
            continue
        r.shuffle(free)
        n = 1 + int(r.integers(min(len(free) - 1, 12)))
        pos = free[:n]
        st = O.State(cells, O.static_field(cells), pos[:, 1].astype(np.int32), pos[:, 0].astype(np.int32), v)
        for i in range(n):
            assert st.candidates(i) == brute_candidates(st, i)


def test_candidates_narrow_periodic_dedupe():  # tests/test_planning.cpp:114-123
    rows = ["######", "......", "......", "......", "######"]
    st = state(rows, [(2, 2)], 4, boundary=1)
    c = st.candidates(0)
    assert len(c) == 18
    assert c == sorted(set(c), key=lambda p: (p[1], p[0]))
    assert c == brute_candidates(st, 0)


def test_two_candidate_closed_form_weights():  # tests/test_planning.cpp:178-186
    st = state(["#####", "#..E#", "#####"], [(1, 1)], 1)
    w, cx, cy = st.weights(0, 1.2)
    assert list(zip(cx, cy)) == [(1, 1), (2, 1)]
    assert w[0] == 1.0 and w[1] == math.exp(1.2)


def test_zero_exit_uniform_weights():  # tests/test_planning.cpp:188-195
    st = state(["#####", "#...#", "#...#", "#...#", "#####"], [(2, 2)], 1)
    assert not np.isfinite(st.field[2, 2])
    w, _, _ = st.weights(0, 1.2)
    assert len(w) == 9 and (w == 1.0).all()


def test_unreachable_candidate_zero_weight():  # tests/test_planning.cpp:197-206
    st = state(["#####", "#E#.#", "##..#", "#...#", "#####"], [(1, 1)], 1)
    assert st.candidates(0) == [(1, 1), (2, 2)]
    w, _, _ = st.weights(0, 1.2)
    assert w[1] == 0.0
    for t in range(2000):
        st.step = t
        st.plan(1.2, 1)
        assert (st.dx[0], st.dy[0]) == (1, 1)


def test_walled_in_agent_stays():  # tests/test_planning.cpp:157-165
    st = state(["###", "#.#", "###"], [(1, 1)], 3)
    for t in range(100):
        st.step = t
        st.plan(1.2, 1)
        assert (st.dx[0], st.dy[0]) == (1, 1)


def test_drive_x_segment_dx():  # tests/test_planning.cpp:243-252 (potential_drop = g * segment_dx)
    L = O.lib()
    assert L.orc_segment_dx(5, 1, 4, 0) == 1
    assert L.orc_segment_dx(5, 1, 0, 4) == -1
    assert L.orc_segment_dx(5, 1, 1, 3) == 2
    assert L.orc_segment_dx(5, 1, 2, 2) == 0


def linear_scan_field(cells, boundary=0):
    """Brute-force Dijkstra picking the cheapest unsettled cell (tests/test_support.hpp:25-71)."""
    h, w = cells.shape
    inf = math.inf
    d = np.full((h, w), inf)
    d[cells == EXIT] = 0.0
    settled = np.zeros((h, w), bool)
    r2 = math.sqrt(2.0)
    while True:
        m = np.where(settled | ~np.isfinite(d), inf, d)
        k = int(np.argmin(m))
        if not np.isfinite(m.flat[k]):
            break
        cy, cx = divmod(k, w)
        settled[cy, cx] = True
        for oy in (-1, 0, 1):
            for ox in (-1, 0, 1):
                if ox == 0 and oy == 0:
                    continue
                ny = cy + oy
                if ny < 0 or ny >= h:
                    continue
                nx = cx + ox
                if boundary:
                    nx %= w
                elif nx < 0 or nx >= w:
                    continue
                if cells[ny, nx] == WALL:
                    continue
                if ox and oy:
                    sx = (cx + ox) % w if boundary else cx + ox
                    if cells[cy, sx] == WALL and cells[ny, cx] == WALL:
                        continue
                nd = d[cy, cx] + (r2 if ox and oy else 1.0)
                if nd < d[ny, nx]:
                    d[ny, nx] = nd
    return d


def test_field_vs_linear_scan_oracle():  # tests/acceptance.cpp:200-219 (1e-9 tolerance)
    r = np.random.default_rng(0xF1E1D)
    for _ in range(12):
        cells = random_grid(r, 20, 20, 0.20, 1 + int(r.integers(5)))
        f = O.static_field(cells)
        want = linear_scan_field(cells)
        both_inf = np.isinf(f) & np.isinf(want)
        assert (both_inf | (np.abs(f - want) <= 1e-9)).all()


def test_field_open_room_exact():  # tests/test_world.cpp:131-140 (exact open-room distances)
    cells = from_rows(["#######", "#.....#", "#.....#", "#.....E", "#######"])
    f = O.static_field(cells)
    assert f[3, 6] == 0.0 and f[3, 5] == 1.0 and f[2, 5] == math.sqrt(2.0)
    assert abs(f[1, 1] - (2 * math.sqrt(2.0) + 3)) < 1e-12
    assert np.isinf(f[0, 0])


def test_trace_length_is_chebyshev():  # tests/test_world.cpp:251-263
    tx = np.empty(64, np.int32)
    ty = np.empty(64, np.int32)
    r = np.random.default_rng(3)
    for _ in range(500):
        ax, ay, bx, by = (int(v) for v in r.integers(0, 30, 4))
        n = O.lib().orc_trace(100, 0, ax, ay, bx, by, tx, ty, 64)
        assert n == max(abs(bx - ax), abs(by - ay))
        if n:
            assert (tx[n - 1], ty[n - 1]) == (bx, by)


def test_movement_order_is_a_permutation():
    for n in (0, 1, 2, 7, 1000):
        o = O.movement_order(n, 5, 3)
        assert sorted(o.tolist()) == list(range(n))


def test_spawn_extremes():  # tests/test_scenario_io.cpp:11-49
    cells = from_rows(OPEN7)
    x, y = O.spawn_agents(cells, 0, 1)
    assert len(x) == 0
    nfree = int((cells == FREE).sum())
    x, y = O.spawn_agents(cells, nfree, 7)
    assert len(set(zip(x.tolist(), y.tolist()))) == nfree
    with pytest.raises(RuntimeError):
        O.spawn_agents(cells, nfree + 1, 7)
