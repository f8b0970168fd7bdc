"""TEST INFRASTRUCTURE -- the checker side's copy of the five synthetic BASELINE.json workloads.

bench.py's reference arm and the full-size fixture generator (tests/golden/make_fullsize.py)
must not import the product package (paper_0911_2900_b200), so the geometry generators of
SURVEY.md 8(d) are restated here in numpy, and the rosters come from the REFERENCE's own
spawn_agents (scenario_io.hpp:47-69, compiled into oracle/_ref) when it is present, else from
the C restatement (oracle/oracle.c, pinned to it by tests/test_oracle_vs_reference.py).
tests/test_configs.py checks that these generators and the product's scenarios.py produce the
same cells and rosters.

The reference publishes no benchmark geometry; these seeded stand-ins have the
configs' shapes, sizes and densities.  All randomness is the reference's counter RNG
(rng.hpp:13-27) on dedicated streams.
"""
from __future__ import annotations

import numpy as np

FREE, WALL, EXIT = 0, 1, 2
CLOSED, PERIODIC_X = 0, 1
EXIT_DISTANCE, DRIVE_X = 0, 1
STREAM_RECT = (1 << 63) + 2      # config 5 rectangles
STREAM_BLOCK = (1 << 63) + 3     # config 3 per-block densities and placement


def rng_u64_np(seed, agent, step, draw) -> np.ndarray:
    """rng_u64 (rng.hpp:13-27), vectorised with wrapping uint64 arithmetic."""
    with np.errstate(over="ignore"):
        s = np.uint64(seed)
        a = np.asarray(agent, np.uint64)
        t = np.asarray(step, np.uint64)
        d = np.asarray(draw, np.uint64)
        z = s ^ (a * np.uint64(0x9E3779B97F4A7C15)) ^ (t * np.uint64(0xBF58476D1CE4E5B9)) ^ \
            (d * np.uint64(0x94D049BB133111EB))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


class Config:
    """One workload: cells (H x W u8), boundary, potential, roster (x, y, v_max), run params."""

    def __init__(self, name, cells, boundary, x, y, v, potential=EXIT_DISTANCE, drive_gradient=0.0,
                 k_s=1.2, seed=1, steps=396):
        self.name, self.cells, self.boundary = name, cells, boundary
        self.x = np.ascontiguousarray(x, np.int32)
        self.y = np.ascontiguousarray(y, np.int32)
        self.v = np.ascontiguousarray(v, np.int32)
        self.potential, self.drive_gradient = potential, drive_gradient
        self.k_s, self.seed, self.steps = k_s, seed, steps

    @property
    def n(self):
        return len(self.x)


def spawn(cells: np.ndarray, n: int, seed: int, boundary: int = CLOSED):
    """spawn_agents (scenario_io.hpp:47-69): the reference's own when oracle/_ref is built."""
    import oracle as O
    if O.have_reference():
        import ctypes as C
        h, w = cells.shape
        x = np.empty(max(n, 1), np.int32)
        y = np.empty(max(n, 1), np.int32)
        c = np.ascontiguousarray(cells, np.uint8).ravel()
        if O.ref().ref_spawn_agents(w, h, c, boundary, n, 4, seed, x, y) != 0:
            raise RuntimeError(O.ref().ref_last_error().decode())
        return x[:n], y[:n]
    x, y = O.spawn_agents(cells, n, seed)
    return np.asarray(x, np.int32), np.asarray(y, np.int32)


def _closed(w, h):
    c = np.zeros((h, w), np.uint8)
    c[0, :] = WALL
    c[-1, :] = WALL
    c[:, 0] = WALL
    c[:, -1] = WALL
    return c


def corridor(seed=1, n=2000, v=4):
    """Config 1: closed 250x50, full-height exit column on the east wall."""
    c = _closed(250, 50)
    c[1:-1, -1] = EXIT
    x, y = spawn(c, n, seed)
    return Config("corridor250x50", c, CLOSED, x, y, np.full(n, v), seed=seed)


def room(seed=1, n=40000, v=4):
    """Config 2: closed 1000x1000, one 10-cell exit mid east wall."""
    c = _closed(1000, 1000)
    c[495:505, -1] = EXIT
    x, y = spawn(c, n, seed)
    return Config("room1000", c, CLOSED, x, y, np.full(n, v), seed=seed)


def ring(seed=1, n=182000, v=4, drive_gradient=1.0):
    """Config 3: periodic-x 4000x200, DriveX, 160 blocks of 10 m with densities U(0.5, 4)
    apportioned to n agents, uniform free cells inside each block."""
    W, H = 4000, 200
    c = np.zeros((H, W), np.uint8)
    c[0, :] = WALL
    c[-1, :] = WALL
    blocks, bw = 160, 25
    u = (rng_u64_np(seed, STREAM_BLOCK, 0, np.arange(blocks)) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    rho = 0.5 + 3.5 * u
    share = rho / rho.sum() * n
    counts = np.floor(share).astype(np.int64)
    rem = n - counts.sum()
    order = np.argsort(-(share - counts), kind="stable")
    counts[order[:rem]] += 1
    rows = np.arange(1, H - 1)
    xs, ys = [], []
    for b in range(blocks):
        k = int(counts[b])
        cand = (rows[:, None] * W + (b * bw + np.arange(bw))[None, :]).ravel().copy()
        F = len(cand)
        draws = rng_u64_np(seed, STREAM_BLOCK, b + 1, np.arange(k))
        for i in range(k):  # partial Fisher-Yates, the spawn_agents rule per block
            j = i + int(draws[i] % np.uint64(F - i))
            cand[i], cand[j] = cand[j], cand[i]
        xs.append(cand[:k] % W)
        ys.append(cand[:k] // W)
    return Config("ring4000x200", c, PERIODIC_X, np.concatenate(xs), np.concatenate(ys), np.full(n, v),
                  DRIVE_X, drive_gradient, seed=seed)


def plaza_cells(width=20000, height=5000, exits=8):
    """make_plaza (scenario_io.hpp:74-105) generalised to W != H: exits at
    (2k+1)*|ring|/(2*exits) along the clockwise non-corner perimeter ring from (1, 0)."""
    w, h = width, height
    c = _closed(w, h)
    L = 2 * (w - 2) + 2 * (h - 2)
    for k in range(exits):
        t = (2 * k + 1) * L // (2 * exits)
        if t < w - 2:
            x, y = 1 + t, 0
        elif t < (w - 2) + (h - 2):
            x, y = w - 1, 1 + t - (w - 2)
        elif t < 2 * (w - 2) + (h - 2):
            x, y = w - 2 - (t - (w - 2) - (h - 2)), h - 1
        else:
            x, y = 0, h - 2 - (t - 2 * (w - 2) - (h - 2))
        c[y, x] = EXIT
    return c


def plaza(seed=1, n=1_000_000, v=4, width=20000, height=5000, exits=8):
    """Config 4: closed 20000x5000 plaza, 8 single-cell perimeter exits."""
    c = plaza_cells(width, height, exits)
    x, y = spawn(c, n, seed)
    return Config("plaza%dx%d" % (width, height), c, CLOSED, x, y, np.full(n, v), seed=seed)


def obstacle_cells(seed=1, width=40000, height=10000, wall_frac=0.15):
    """Config 5 geometry: seeded rectangles (sides 2..40) until >= wall_frac of cells are Wall,
    four ten-cell exits mid-side with the cell inside each kept Free."""
    W, H = width, height
    c = _closed(W, H)
    walls = int(2 * W + 2 * H - 4)
    target = int(np.ceil(wall_frac * W * H))
    k = 0
    while walls < target:
        batch = rng_u64_np(seed, STREAM_RECT, k // 1024, np.arange(4 * 1024)).reshape(1024, 4)
        for r in batch:
            if walls >= target:
                break
            w = 2 + int(r[0] % np.uint64(39))
            h = 2 + int(r[1] % np.uint64(39))
            x0 = 1 + int(r[2] % np.uint64(max(W - 2 - w, 1)))
            y0 = 1 + int(r[3] % np.uint64(max(H - 2 - h, 1)))
            sub = c[y0:y0 + h, x0:x0 + w]
            walls += int(np.count_nonzero(sub != WALL))
            sub[...] = WALL
            k += 1
    mx, my = W // 2 - 5, H // 2 - 5
    c[0, mx:mx + 10] = EXIT
    c[1, mx:mx + 10] = FREE
    c[H - 1, mx:mx + 10] = EXIT
    c[H - 2, mx:mx + 10] = FREE
    c[my:my + 10, 0] = EXIT
    c[my:my + 10, 1] = FREE
    c[my:my + 10, W - 1] = EXIT
    c[my:my + 10, W - 2] = FREE
    return c


def obstacles(seed=1, n=10_000_000, width=40000, height=10000, wall_frac=0.15):
    """Config 5: mixed v_max = 2 + rng_u64(seed, id, 0, 1) % 4, set after spawning."""
    c = obstacle_cells(seed, width, height, wall_frac)
    x, y = spawn(c, n, seed)
    v = 2 + (rng_u64_np(seed, np.arange(n, dtype=np.uint64), 0, 1) % np.uint64(4))
    return Config("obstacles%dx%d" % (width, height), c, CLOSED, x, y, v.astype(np.int32), seed=seed)


CONFIGS = {"corridor": corridor, "room": room, "ring": ring, "plaza": plaza, "obstacles": obstacles}


def build(name: str, **kw) -> Config:
    return CONFIGS[name](**kw)


def roster_digest(x, y, v) -> str:
    """sha256 of the roster arrays (fixtures pin the initial state with it)."""
    import hashlib
    h = hashlib.sha256()
    for a in (x, y, v):
        h.update(np.ascontiguousarray(a, np.int32).tobytes())
    return h.hexdigest()


def cells_digest(cells) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(cells, np.uint8).tobytes()).hexdigest()


def desired_digest(dx, dy, mask) -> int:
    """Order-sensitive 64-bit digest of the desired cells of the agents in `mask` (the agents
    alive entering a step): sum over i of ((dx_i * 1000003 + dy_i) ^ (i * phi64)) mod 2^64."""
    idx = np.flatnonzero(mask).astype(np.uint64)
    with np.errstate(over="ignore"):
        a = np.asarray(dx, np.int64)[idx].astype(np.uint64) * np.uint64(1000003) + \
            np.asarray(dy, np.int64)[idx].astype(np.uint64)
        return int(np.sum(a ^ (idx * np.uint64(0x9E3779B97F4A7C15)), dtype=np.uint64))
