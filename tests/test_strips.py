"""x-strip decomposition of the planning phase (multi-GPU path).

GPU: contexts playing the ranks plan their strips (fp_plan_strip); the element-wise sum of their
desired-cell arrays equals the full plan_phase bit for bit, and a simulation stepped that way
(combine, then the replicated motion) stays identical to the single-context run.
CPU (gloo, world_size 2): the same decomposition through torch.distributed, with the C
restatement standing in for each rank's planning kernel."""
import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_0911_2900_b200.dist import strip_bounds
from tests.helpers import random_grid, random_periodic


def test_strips_tile_the_grid():
    for W in (1, 7, 250, 20000):
        for world in (1, 2, 3, 4, 8):
            if world > W:
                continue
            b = [strip_bounds(W, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == W
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert all(lo < hi for lo, hi in b)


def _scenario(periodic):
    rng = np.random.default_rng(99 if periodic else 98)
    cells = random_periodic(rng, 60, 20, 0.05) if periodic else random_grid(rng, 60, 40, 0.06, 3)
    boundary = 1 if periodic else 0
    x, y = O.spawn_agents(cells, 500, 5)
    return cells, boundary, np.asarray(x, np.int32), np.asarray(y, np.int32)


@pytest.mark.gpu
@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_strip_plans_sum_to_the_full_plan_and_trajectory(periodic, world):
    from paper_0911_2900_b200 import fastped as fp
    cells, boundary, x, y = _scenario(periodic)
    grid = fp.Grid(cells, 0.4, boundary)
    ro = lambda: fp.Roster(x.copy(), y.copy(), np.full(len(x), 4, np.int32), np.ones(len(x), np.uint8))  # noqa: E731
    full = fp.SimState(grid, None, ro())
    ranks = [fp.SimState(grid, None, ro()) for _ in range(world)]
    bounds = [strip_bounds(grid.width, r, world) for r in range(world)]
    p = fp.SimParams(k_s=1.2, seed=17, steps=1)
    for s in range(15):
        fp.plan_phase(full, p)
        fdx, fdy = full.desired()
        sdx = np.zeros_like(fdx)
        sdy = np.zeros_like(fdy)
        for st, (lo, hi) in zip(ranks, bounds):
            st.plan_strip(p.k_s, p.seed, lo, hi)
            dx, dy = st.desired()
            sdx += dx
            sdy += dy
        al = full.agents()[2].astype(bool)
        assert np.array_equal(sdx[al], fdx[al]) and np.array_equal(sdy[al], fdy[al]), s
        fo = fp.move_phase(full, p)
        full.step = full.step + 1
        for st in ranks:  # what the all-reduce delivers, then the replicated motion
            st.set_desired(sdx, sdy)
            o = fp.move_phase(st, p)
            st.step = st.step + 1
            assert o.exited == fo.exited and o.displacement_cells == fo.displacement_cells
            assert fp.state_hash(st) == fp.state_hash(full)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cells, boundary, x, y = _scenario(False)
    field = O.static_field(cells, boundary)
    lo, hi = strip_bounds(cells.shape[1], rank, world)
    st = O.State(cells, field, x, y, 4, boundary=boundary)
    ok = True
    for s in range(8):
        st.plan(1.2, 17)  # stand-in for this rank's plan kernel: keep only the strip's agents
        mine = (st.x >= lo) & (st.x < hi) & st.alive.astype(bool)
        dx = torch.from_numpy(np.where(mine, st.dx, 0).astype(np.int32))
        dy = torch.from_numpy(np.where(mine, st.dy, 0).astype(np.int32))
        dist.all_reduce(dx)
        dist.all_reduce(dy)
        ref = O.State(cells, field, st.x.copy(), st.y.copy(), 4, alive=st.alive.copy(), boundary=boundary,
                      step=st.step)
        ref.plan(1.2, 17)
        al = st.alive.astype(bool)
        ok &= bool(np.array_equal(dx.numpy()[al], ref.dx[al]) and np.array_equal(dy.numpy()[al], ref.dy[al]))
        st.dx[:] = dx.numpy()
        st.dy[:] = dy.numpy()
        st.move(17)
        st.step = st.step + 1
    q.put((rank, ok, st.hash()))
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_two_rank_strip_decomposition_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    for p_ in procs:
        p_.join(150)
        assert p_.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert all(ok for _, ok, _ in res)
    assert res[0][2] == res[1][2]  # both ranks hold the same state
    cells, boundary, x, y = _scenario(False)
    single = O.State(cells, O.static_field(cells, boundary), x, y, 4, boundary=boundary)
    for _ in range(8):
        single.step_once(1.2, 17)
    assert res[0][2] == single.hash()
