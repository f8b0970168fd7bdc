"""Synthetic stand-ins for BASELINE.json's five configurations.

The reference publishes no benchmark geometry; these seeded generators supply
grids and rosters with the configs' shapes, sizes and densities.  All randomness comes from the
reference's own counter RNG (rng.hpp:21-27) on dedicated streams, so every roster is a pure
function of (config, seed) and is fed identically to the CUDA engine and to the CPU checkers.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import fastped as fp

STREAM_RECT = (1 << 63) + 2      # config 5 rectangles
STREAM_BLOCK = (1 << 63) + 3     # config 3 per-block densities and placement


def rng_u64_np(seed, agent, step, draw) -> np.ndarray:
    """Vectorised rng_u64 (rng.hpp:13-27) with wrapping uint64 arithmetic."""
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


@dataclass
class Workload:
    name: str
    grid: fp.Grid
    roster: fp.Roster
    potential: int = fp.EXIT_DISTANCE
    drive_gradient: float = 0.0
    k_s: float = 1.2
    seed: int = 1
    steps: int = 396


def corridor(seed: int = 1, n: int = 2000, v: int = 4) -> Workload:
    """Config 1: closed 250x50, walls N/S/W, full-width exit on the east wall."""
    W, H = 250, 50
    cells = np.zeros((H, W), np.uint8)
    cells[0, :] = fp.WALL
    cells[-1, :] = fp.WALL
    cells[:, 0] = fp.WALL
    cells[:, -1] = fp.WALL
    cells[1:-1, -1] = fp.EXIT
    g = fp.Grid(cells)
    return Workload("corridor250x50", g, fp.spawn_agents(g, n, v, seed), seed=seed)


def room(seed: int = 1, n: int = 40000, v: int = 4) -> Workload:
    """Config 2: closed 1000x1000, one 10-cell exit mid east wall."""
    W = H = 1000
    cells = np.zeros((H, W), np.uint8)
    cells[0, :] = fp.WALL
    cells[-1, :] = fp.WALL
    cells[:, 0] = fp.WALL
    cells[:, -1] = fp.WALL
    cells[495:505, -1] = fp.EXIT
    g = fp.Grid(cells)
    return Workload("room1000", g, fp.spawn_agents(g, n, v, seed), seed=seed)


def ring(seed: int = 1, n: int = 182000, v: int = 4, drive_gradient: float = 1.0) -> Workload:
    """Config 3: periodic-x 4000x200 corridor, DriveX potential (S = -g*x), 160 blocks of 10 m
    with per-block densities U(0.5, 4) /m^2 apportioned to n agents in total."""
    W, H = 4000, 200
    cells = np.zeros((H, W), np.uint8)
    cells[0, :] = fp.WALL
    cells[-1, :] = fp.WALL
    g = fp.Grid(cells, 0.4, fp.PERIODIC_X)
    blocks, bw = 160, 25
    u = (rng_u64_np(seed, STREAM_BLOCK, 0, np.arange(blocks)) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    rho = 0.5 + 3.5 * u
    share = rho / rho.sum() * n
    counts = np.floor(share).astype(np.int64)
    rem = n - counts.sum()
    order = np.argsort(-(share - counts), kind="stable")
    counts[order[:rem]] += 1
    free_rows = np.arange(1, H - 1)
    xs, ys = [], []
    for b in range(blocks):
        c = int(counts[b])
        cand = (free_rows[:, None] * W + (b * bw + np.arange(bw))[None, :]).ravel()  # row-major
        F = len(cand)
        draws = rng_u64_np(seed, STREAM_BLOCK, b + 1, np.arange(c))
        cand = cand.copy()
        for i in range(c):  # partial Fisher-Yates (the spawn_agents rule, per block)
            j = i + int(draws[i] % np.uint64(F - i))
            cand[i], cand[j] = cand[j], cand[i]
        xs.append(cand[:c] % W)
        ys.append(cand[:c] // W)
    x = np.concatenate(xs).astype(np.int32)
    y = np.concatenate(ys).astype(np.int32)
    r = fp.Roster(x, y, np.full(n, v, np.int32), np.ones(n, np.uint8))
    return Workload("ring4000x200", g, r, fp.DRIVE_X, drive_gradient, seed=seed)


def plaza(seed: int = 1, n: int = 1_000_000, v: int = 4, width: int = 20000, height: int = 5000,
          exits: int = 8) -> Workload:
    """Config 4: closed 20000x5000 plaza, 8 single-cell perimeter exits (make_plaza's rule)."""
    g = fp.make_plaza(0.4 * width, exits, 0.4, width=width, height=height)
    return Workload("plaza%dx%d" % (width, height), g, fp.spawn_agents(g, n, v, seed), seed=seed)


def obstacles(seed: int = 1, n: int = 10_000_000, width: int = 40000, height: int = 10000,
              wall_frac: float = 0.15) -> Workload:
    """Config 5: closed 40000x10000, seeded rectangles (sides 2..40) until >= 15% of cells are
    Wall, 4 ten-cell exits mid-side, mixed v_max = 2 + rng_u64(seed, id, 0, 1) % 4."""
    W, H = width, height
    cells = np.zeros((H, W), np.uint8)
    cells[0, :] = fp.WALL
    cells[-1, :] = fp.WALL
    cells[:, 0] = fp.WALL
    cells[:, -1] = fp.WALL
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
            sub = cells[y0:y0 + h, x0:x0 + w]
            walls += int(np.count_nonzero(sub != fp.WALL))
            sub[...] = fp.WALL
            k += 1
    # four ten-cell exits at mid-sides, with the cells inside them kept Free
    mx, my = W // 2 - 5, H // 2 - 5
    for xs, ys, ix, iy in ((slice(mx, mx + 10), 0, 0, 1), (slice(mx, mx + 10), H - 1, 0, -1)):
        cells[ys, xs] = fp.EXIT
        cells[ys + iy, xs] = fp.FREE
    for ys, xs, ix in ((slice(my, my + 10), 0, 1), (slice(my, my + 10), W - 1, -1)):
        cells[ys, xs] = fp.EXIT
        cells[ys, xs + ix] = fp.FREE
    g = fp.Grid(cells)
    r = fp.spawn_agents(g, n, 4, seed)
    r.v_max = (2 + (rng_u64_np(seed, np.arange(n, dtype=np.uint64), 0, 1) % np.uint64(4))).astype(np.int32)
    return Workload("obstacles%dx%d" % (W, H), g, r, seed=seed)


CONFIGS = {
    "corridor": corridor,   # BASELINE.json configs[0]
    "room": room,           # configs[1]
    "ring": ring,           # configs[2]
    "plaza": plaza,         # configs[3]
    "obstacles": obstacles, # configs[4]
}


def build(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)
