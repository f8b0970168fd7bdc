"""Shared fixtures for the parity tests: seeded random scenarios fed identically to the CUDA
engine (paper_0911_2900_b200.fastped) and to the CPU checkers (oracle/)."""
from __future__ import annotations

import numpy as np

FREE, WALL, EXIT = 0, 1, 2


def from_rows(rows):
    t = {"#": WALL, "E": EXIT}
    return np.array([[t.get(c, FREE) for c in r] for r in rows], np.uint8)


def random_grid(rng: np.random.Generator, w: int, h: int, wall_frac: float, exits: int) -> np.ndarray:
    """Closed grid: Wall border, ~wall_frac interior walls, `exits` exits on the border
    (the shape of tests/test_support.hpp:95-117; our own seeded generator)."""
    c = np.zeros((h, w), np.uint8)
    c[rng.random((h, w)) < wall_frac] = WALL
    c[0, :] = WALL
    c[-1, :] = WALL
    c[:, 0] = WALL
    c[:, -1] = WALL
    for _ in range(exits):
        side = rng.integers(4)
        if side == 0:
            c[0, rng.integers(1, w - 1)] = EXIT
        elif side == 1:
            c[h - 1, rng.integers(1, w - 1)] = EXIT
        elif side == 2:
            c[rng.integers(1, h - 1), 0] = EXIT
        else:
            c[rng.integers(1, h - 1), w - 1] = EXIT
    return c


def random_periodic(rng: np.random.Generator, w: int, h: int, wall_frac: float) -> np.ndarray:
    c = np.zeros((h, w), np.uint8)
    c[rng.random((h, w)) < wall_frac] = WALL
    c[0, :] = WALL
    c[-1, :] = WALL
    return c


def spawn(cells: np.ndarray, n: int, seed: int):
    import oracle
    return oracle.spawn_agents(cells, n, seed)
