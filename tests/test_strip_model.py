"""The x-strip decomposition ALGORITHM of strip.cu, restated in Python and run as a real
world_size-2 torch.distributed job (gloo, CPU) -- the host-side logic of the multi-GPU path:

  * each rank owns the agents standing in its columns and keeps ONLY its window
    [x_lo - 5, x_hi + 5) of the occupancy (cells outside are "unknown" and must never be read);
  * walks whose footprint touches a band (5 cells either side of a shared strip edge), closed
    under shared footprint cells, are deferred; the rest walk locally in reference order;
  * one allgather per step carries the deferred records (with the snapshot occupancy of their
    footprint cells) and the local exits; every rank resolves the deferred walks in rank order
    and applies the results inside its window, ownership following the final cell.

Every step each rank checks, against the sequential oracle (oracle/oracle.c, pinned to the
reference) run in the same process: the exit list in processing order, the displacement, the
positions of the agents it owns, and its whole window of occupancy.  The GPU implementation
(tests/test_strips.py) is held to the same equalities through the C ABI.
"""
import os
import socket

import numpy as np
import pytest

import oracle as O
from tests.helpers import random_grid, random_periodic

WALL, EXIT = 1, 2
K_S, SEED = 1.2, 21


def segment_dx(W, periodic, ax, bx):  # world.hpp:125-132
    d = bx - ax
    if periodic:
        alt = d - W if d > 0 else d + W
        if abs(alt) < abs(d):
            d = alt
    return d


def bresenham(W, periodic, ax, ay, bx, by):  # world.hpp:143-167, a exclusive, b inclusive
    tx = ax + segment_dx(W, periodic, ax, bx)
    dx, sx = abs(tx - ax), (1 if ax < tx else -1)
    dy, sy = -abs(by - ay), (1 if ay < by else -1)
    err, x, y, out = dx + dy, ax, ay, []
    while not (x == tx and y == by):
        e2 = 2 * err
        if e2 >= dy:
            err += dy
            x += sx
        if e2 <= dx:
            err += dx
            y += sy
        out.append((x % W if periodic else x, y))
    return out


class Rank:
    def __init__(self, cells, periodic, truth, rank, nranks):
        self.cells, self.periodic = cells, periodic
        self.H, self.W = cells.shape
        self.rank, self.nranks = rank, nranks
        self.lo, self.hi = rank * self.W // nranks, (rank + 1) * self.W // nranks
        x, y, a = truth.x, truth.y, truth.alive.astype(bool)
        self.x, self.y = x.copy(), y.copy()
        self.alive = a.copy()
        self.owned = a & (x >= self.lo) & (x < self.hi)
        self.occ = np.full((self.H, self.W), -1, np.int8)  # -1: outside the window (unknown)
        win = self.window_cols()
        self.occ[:, win] = 0
        for i in np.flatnonzero(a):
            if self.in_window(x[i]):
                self.occ[y[i], x[i]] = 1

    def window_cols(self):
        cols = [(c % self.W) if self.periodic else c for c in range(self.lo - 5, self.hi + 5)]
        return [c for c in cols if 0 <= c < self.W]

    def in_window(self, x):
        d = x - (self.lo - 5)
        if self.periodic:
            d %= self.W
        return 0 <= d < (self.hi - self.lo) + 10

    def in_band(self, x):
        if self.nranks < 2:
            return False
        edges = []
        if self.periodic or self.lo > 0:
            edges.append(self.lo)
        if self.periodic or self.hi < self.W:
            edges.append(self.hi % self.W if self.periodic else self.hi)
        for e in edges:
            d = x - e
            if self.periodic:
                d = (d + self.W // 2) % self.W - self.W // 2
            if -5 <= d < 5:
                return True
        return False

    def read(self, x, y):
        v = self.occ[y, x]
        assert v >= 0, f"rank {self.rank} read cell ({x},{y}) outside its window"
        return bool(v)

    def record(self, i, tx, ty, v):
        sx, sy = int(self.x[i]), int(self.y[i])
        path, ex = [], False
        for (cx, cy) in bresenham(self.W, self.periodic, sx, sy, tx, ty)[:v]:
            if self.cells[cy, cx] == WALL:
                break
            path.append((cx, cy))
            if self.cells[cy, cx] == EXIT:
                ex = True
                break
        exit_free = ex and not self.read(*path[-1])
        mf = len(path) - (1 if exit_free else 0)
        return dict(id=i, start=(sx, sy), path=path, exit=ex, fp=[(sx, sy)] + path[:mf])

    def step(self, desired_x, desired_y, v_max, rank_of, allgather):
        recs = []
        for i in np.flatnonzero(self.owned & self.alive):
            r = self.record(i, int(desired_x[i]), int(desired_y[i]), int(v_max[i]))
            if r["path"]:
                recs.append(r)
        # deferral: band seeds, closed under shared footprint cells
        defer = {r["id"] for r in recs if any(self.in_band(c[0]) for c in r["fp"])}
        cells = set(c for r in recs if r["id"] in defer for c in r["fp"])
        changed = True
        while changed:
            changed = False
            for r in recs:
                if r["id"] not in defer and any(c in cells for c in r["fp"]):
                    defer.add(r["id"])
                    cells.update(r["fp"])
                    changed = True
        # local walks in the reference order
        hops, exits = 0, []
        for r in sorted((r for r in recs if r["id"] not in defer), key=lambda r: rank_of[r["id"]]):
            h = self.walk(r, self.read, self.write)
            hops += h[0]
            if h[1]:
                exits.append((rank_of[r["id"]], r["id"]))
        # exchange: deferred records with the snapshot occupancy of their cells, local exits
        mine = [dict(r, rank=rank_of[r["id"]], occ={c: self.read(*c) for c in [r["start"]] + r["path"]})
                for r in recs if r["id"] in defer]
        parts = allgather((mine, exits, hops))
        self.n_deferred = sum(len(p[0]) for p in parts)
        allrec = sorted((r for p in parts for r in p[0]), key=lambda r: r["rank"])
        occ = {}
        for r in allrec:
            for c, o in r["occ"].items():
                occ[c] = occ.get(c, False) or o
        rexits, rhops = [], 0
        for r in allrec:  # every rank resolves the union in rank order
            h = self.walk(r, lambda x, y: occ[(x, y)], lambda x, y, val: occ.__setitem__((x, y), val), track=True)
            rhops += h[0]
            if h[1]:
                rexits.append((r["rank"], r["id"]))
        for (cx, cy), o in occ.items():
            if self.in_window(cx):
                self.occ[cy, cx] = 1 if o else 0
        all_exits = sorted([e for p in parts for e in p[1]] + rexits)
        for _, i in all_exits:
            self.alive[i] = False
        return all_exits, sum(p[2] for p in parts) + rhops

    def write(self, x, y, val):
        assert self.occ[y, x] >= 0, f"rank {self.rank} wrote cell ({x},{y}) outside its window"
        self.occ[y, x] = 1 if val else 0

    def walk(self, r, read, write, track=False):  # engine.hpp:113-133 on the given occupancy
        h = 0
        while h < len(r["path"]) and not read(*r["path"][h]):
            h += 1
        exited = h == len(r["path"]) and r["exit"] and h > 0
        i = r["id"]
        if h:
            write(*r["start"], False)
            fx, fy = r["path"][h - 1]
            self.x[i], self.y[i] = fx, fy
            if not exited:
                write(fx, fy, True)
        if track:  # ownership follows the final cell (only deferred walks cross an edge)
            self.owned[i] = (not exited) and self.lo <= self.x[i] < self.hi
        return h, exited


def scenario(periodic):
    rng = np.random.default_rng(7 if periodic else 8)
    if periodic:
        cells = random_periodic(rng, 48, 16, 0.05)
    else:
        cells = random_grid(rng, 48, 30, 0.05, 4)
        cells[-1, 22:26] = EXIT  # an exit right at the strip edge (x = 24)
    x, y = O.spawn_agents(cells, 420, 4)
    return cells, np.asarray(x, np.int32), np.asarray(y, np.int32)


def _worker(rank, world, port, periodic, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allgather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    cells, x, y = scenario(periodic)
    v = 1 + (np.arange(len(x)) * 31) % 5
    truth = O.State(cells, O.static_field(cells, int(periodic)), x, y, v, boundary=int(periodic))
    me = Rank(cells, periodic, truth, rank, world)
    ok, deferred, crossings = True, 0, 0
    for _ in range(30):
        before = me.owned.copy()
        alive_ids = np.flatnonzero(truth.alive)
        perm = O.movement_order(len(alive_ids), SEED, truth.step)
        rank_of = {int(alive_ids[p]): k for k, p in enumerate(perm)}
        truth.plan(K_S, SEED)  # planning reads only balls inside the window (checked below)
        exits, disp = me.step(truth.dx, truth.dy, truth.v_max, rank_of, allgather)
        tex, tdisp = truth.move(SEED)
        truth.step = truth.step + 1
        ok &= [i for _, i in exits] == tex.tolist() and disp == tdisp
        own = np.flatnonzero(me.owned & truth.alive.astype(bool))
        ok &= bool(np.array_equal(me.x[own], truth.x[own]) and np.array_equal(me.y[own], truth.y[own]))
        tocc = (truth.occ.reshape(cells.shape) >= 0).astype(np.int8)
        win = me.window_cols()
        ok &= bool(np.array_equal(me.occ[:, win], tocc[:, win]))
        owners = allgather(me.owned & truth.alive.astype(bool))
        ok &= bool((np.sum(owners, 0) == truth.alive.astype(int)).all())  # each alive agent: one owner
        deferred += me.n_deferred
        crossings += int((before & ~me.owned & truth.alive.astype(bool)).sum())
    q.put((rank, ok, deferred, crossings))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.timeout(300)
@pytest.mark.parametrize("periodic", [False, True])
def test_strip_algorithm_two_ranks_gloo(periodic):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, periodic, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    for p_ in procs:
        p_.join(280)
        assert p_.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert all(r[1] for r in res)
    assert res[0][2] > 0 and sum(r[3] for r in res) > 0  # walks were deferred and agents changed strips
