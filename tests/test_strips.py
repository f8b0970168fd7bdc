"""Multi-GPU x-strip decomposition of one simulation (strip.cu).

GPU: N contexts on one device play the ranks (virtual strips, fp_strips_step / fp_strips_run --
the in-process transport); every step's merged state, exit list (processing order), alive
count and displacement must equal the single-context run, which tests/test_fullsize_golden.py
pins to the reference.  Cases cover closed and periodic grids, mixed v_max, an exit queue cut by
a strip edge, strips narrower than the 5-cell band, and the full-size configs 3-5.  The host
transport (a Python allgather over gloo) runs two processes on the one GPU.
CPU: strip bounds; the gloo world_size-2 test of the decomposition algorithm itself lives in
tests/test_strip_model.py."""
import ctypes as C
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


def test_library_strip_bounds_agree():
    from paper_0911_2900_b200 import fastped as fp
    for W, world in ((250, 3), (20000, 8), (17, 4)):
        for r in range(world):
            assert fp.strip_bounds(W, r, world) == strip_bounds(W, r, world)


def _compare(fp, make_single, make_set, steps, k_s=1.2, seed=17):
    single = make_single()
    ss = make_set()
    p = fp.SimParams(k_s=k_s, seed=seed, steps=1)
    for s in range(steps):
        a = fp.step(single, p)
        b = ss.step(p)
        assert (b.alive, b.exited, b.displacement_cells) == (a.alive, a.exited, a.displacement_cells), s
        buf = np.empty(max(single.n, 1), np.uint32)
        n = C.c_uint32()
        fp._check(fp.library().fp_get_exited(single._ctx, buf, len(buf), C.byref(n)), single._ctx)
        assert ss.exited() == buf[: n.value].tolist(), s
        assert ss.state_hash() == fp.state_hash(single), s
    return single, ss


def _roster(fp, x, y, v):
    return fp.Roster(np.asarray(x, np.int32), np.asarray(y, np.int32), np.asarray(v, np.int32),
                     np.ones(len(x), np.uint8))


@pytest.mark.gpu
@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("world", [2, 3, 5])
def test_virtual_strips_equal_single_gpu(periodic, world):
    from paper_0911_2900_b200 import fastped as fp
    rng = np.random.default_rng(99 if periodic else 98)
    cells = random_periodic(rng, 80, 24, 0.05) if periodic else random_grid(rng, 80, 40, 0.06, 4)
    grid = fp.Grid(cells, 0.4, 1 if periodic else 0)
    x, y = O.spawn_agents(cells, 700, 5)
    v = 1 + (np.arange(len(x)) * 7919) % 5  # mixed v_max 1..5
    _compare(fp, lambda: fp.SimState(grid, None, _roster(fp, x, y, v)),
             lambda: fp.StripSet(grid, None, _roster(fp, x, y, v), world), 40)


@pytest.mark.gpu
def test_exit_queue_cut_by_a_strip_edge():
    """A dense room whose only exit lies on a strip edge: the queue's conflict chains cross the
    edge every step (the deferred set is large and deep)."""
    from paper_0911_2900_b200 import fastped as fp
    W, H = 120, 60
    cells = np.zeros((H, W), np.uint8)
    cells[0, :] = cells[-1, :] = 1
    cells[:, 0] = cells[:, -1] = 1
    cells[-1, 58:63] = 2  # exit on the bottom wall, x = 58..62
    grid = fp.Grid(cells)
    x, y = O.spawn_agents(cells, 3000, 3)
    v = np.full(len(x), 4)
    bounds = [(0, 60), (60, 61), (61, 63), (63, W)]  # strips of 1 and 2 columns around the exit
    _compare(fp, lambda: fp.SimState(grid, None, _roster(fp, x, y, v)),
             lambda: fp.StripSet(grid, None, _roster(fp, x, y, v), 4, x_bounds=bounds), 80)


@pytest.mark.gpu
def test_strips_run_equals_single_run():
    from paper_0911_2900_b200 import fastped as fp
    rng = np.random.default_rng(5)
    cells = random_grid(rng, 200, 90, 0.04, 6)
    grid = fp.Grid(cells)
    x, y = O.spawn_agents(cells, 4000, 9)
    v = np.full(len(x), 4)
    single = fp.SimState(grid, None, _roster(fp, x, y, v))
    ss = fp.StripSet(grid, None, _roster(fp, x, y, v), 4)
    p = fp.SimParams(k_s=1.2, seed=3, steps=60)
    a = fp.run(single, p)
    b = ss.run(p)
    assert (b.exited, b.displacement_cells, b.alive, b.agent_updates) == \
        (a.exited, a.displacement_cells, a.alive, a.agent_updates)
    assert ss.state_hash() == fp.state_hash(single)


@pytest.mark.gpu
@pytest.mark.timeout(1500)
@pytest.mark.parametrize("config,world,steps", [("plaza", 4, 40), ("ring", 4, 40), ("room", 3, 120),
                                                ("obstacles", 3, 4)])
def test_full_size_configs_on_virtual_strips(config, world, steps):
    from paper_0911_2900_b200 import fastped as fp
    from paper_0911_2900_b200 import scenarios
    wl = scenarios.build(config)

    def single():
        st = fp.SimState(wl.grid, None, wl.roster)
        if wl.potential:
            st.set_potential(wl.potential, wl.drive_gradient)
        return st

    def strips():
        ss = fp.StripSet(wl.grid, None, wl.roster, world)
        if wl.potential:
            ss.set_potential(wl.potential, wl.drive_gradient)
        return ss

    _compare(fp, single, strips, steps, wl.k_s, wl.seed)


@pytest.mark.gpu
@pytest.mark.timeout(300)
def test_nccl_transport_single_rank_communicator():
    """The library's own NCCL transport on hardware, as far as one GPU allows: a one-rank
    communicator (fp_nccl_unique_id -> fp_strip_set_nccl -> ncclCommInitRank) whose every step
    runs the real exchange on the context's stream -- ncclAllGather of the headers, the read
    back, ncclGroupStart/End around the (empty) peer loop and the self copy -- and must equal
    the plain single-context run, exits in processing order included.  Two NCCL ranks cannot share
    one device, so the peer sends stay covered by the host and in-process transports."""
    from paper_0911_2900_b200 import fastped as fp
    rng = np.random.default_rng(1234)
    cells = random_grid(rng, 160, 70, 0.05, 5)
    grid = fp.Grid(cells)
    x, y = O.spawn_agents(cells, 2500, 21)
    v = np.full(len(x), 4)
    single = fp.SimState(grid, None, _roster(fp, x, y, v))
    rank = fp.StripRank(grid, None, _roster(fp, x, y, v), 0, 1, 0, nccl_id=fp.nccl_unique_id())
    assert (rank.x_lo, rank.x_hi) == (0, 160) and rank.owned().all()
    p = fp.SimParams(k_s=1.2, seed=29, steps=1)
    for s in range(40):
        a = fp.step(single, p)
        b = fp.step(rank, p)
        assert (b.alive, b.exited, b.displacement_cells) == (a.alive, a.exited, a.displacement_cells), s
        assert fp.state_hash(rank) == fp.state_hash(single), s
    rs_a = fp.run(single, fp.SimParams(k_s=1.2, seed=29, steps=20))
    rs_b = fp.run(rank, fp.SimParams(k_s=1.2, seed=29, steps=20))
    assert (rs_b.alive, rs_b.exited, rs_b.displacement_cells) == (rs_a.alive, rs_a.exited, rs_a.displacement_cells)
    assert fp.state_hash(rank) == fp.state_hash(single)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _host_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_0911_2900_b200 import fastped as fp
    from paper_0911_2900_b200.dist import gather_state, strip_rank
    rng = np.random.default_rng(98)
    cells = random_grid(rng, 80, 40, 0.06, 4)
    grid = fp.Grid(cells)
    x, y = O.spawn_agents(cells, 700, 5)
    st = strip_rank(grid, None, _roster(fp, x, y, np.full(len(x), 4)), 0, transport="host")
    p = fp.SimParams(k_s=1.2, seed=17, steps=1)
    hashes = []
    for _ in range(25):
        fp.step(st, p)
        gx, gy, ga = gather_state(st)
        hashes.append(fp.hash_roster(st.step, st.alive, gx, gy, ga))
    q.put((rank, hashes))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(300)
def test_two_processes_host_transport_gloo():
    """Two ranks, one process each, on the one GPU; the exchange is a gloo allgather on the host
    (the ranks' kernels never wait on each other).  Every step equals the single context."""
    import torch.multiprocessing as mp
    from paper_0911_2900_b200 import fastped as fp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_host_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    for p_ in procs:
        p_.join(250)
        assert p_.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert res[0][1] == res[1][1]
    rng = np.random.default_rng(98)
    cells = random_grid(rng, 80, 40, 0.06, 4)
    x, y = O.spawn_agents(cells, 700, 5)
    single = fp.SimState(fp.Grid(cells), None, _roster(fp, x, y, np.full(len(x), 4)))
    p = fp.SimParams(k_s=1.2, seed=17, steps=1)
    for h in res[0][1]:
        fp.step(single, p)
        assert fp.state_hash(single) == h
