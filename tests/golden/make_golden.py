"""Regenerates the golden fixtures of this directory by running the REFERENCE implementation
itself -- the unmodified headers of /root/reference compiled into oracle/_ref by oracle/Makefile
(`make -C oracle`) -- on small seeded scenarios.  The fixtures pin both the C restatement
(oracle/) and the CUDA engine without needing /root/reference at test time.

    python tests/golden/make_golden.py        # writes tests/golden/*.npz

Each scenario is built from our own seeded generators (tests/helpers.py); nothing here comes
from a third-party benchmark.  Per scenario the fixture stores the grid, the reference's static
field, the initial roster and, for every step, the desired cells of the plan phase, the
movement order, the positions / alive flags after the move phase, the exited ids in
processing order and state_hash.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from tests.helpers import random_grid, random_periodic  # noqa: E402

K_S = 1.2


def scenarios():
    rng = np.random.default_rng(0x601DE7)
    out = []
    # closed room, four exits, light obstacles, v=4 (the headline configuration, shrunk)
    c = random_grid(rng, 48, 32, 0.06, 4)
    out.append(("room_v4", c, 0, 0, 0.0, 260, 4, 30, 11))
    # dense closed corridor with mixed v_max 1..5 and a full-height exit column
    c = random_grid(rng, 64, 20, 0.03, 0)
    c[1:-1, -1] = 2
    out.append(("corridor_mixed_v", c, 0, 0, 0.0, 520, -1, 30, 12))
    # periodic ring under DriveX (no exits, field unused)
    c = random_periodic(rng, 72, 14, 0.05)
    out.append(("ring_drivex", c, 1, 1, 1.0, 300, 4, 25, 13))
    # periodic ring with exits and ExitDistance (wrap-around field and walks)
    c = random_periodic(rng, 40, 16, 0.04)
    c[5, 7] = 2
    c[10, 31] = 2
    out.append(("ring_exitdistance", c, 1, 0, 0.0, 180, 3, 25, 14))
    # enclosed pocket (unreachable agents plan with uniform weights)
    c = random_grid(rng, 30, 30, 0.0, 2)
    c[10:20, 10] = 1
    c[10:20, 19] = 1
    c[10, 10:20] = 1
    c[19, 10:20] = 1
    out.append(("pocket", c, 0, 0, 0.0, 150, 5, 20, 15))
    return out


def roster(cells, n, v, seed):
    x, y = O.spawn_agents(cells, n, seed)
    if v > 0:
        vm = np.full(len(x), v, np.int32)
    else:  # mixed 1..5 from a dedicated rng stream (BASELINE config-5 style)
        vm = np.array([1 + O.rng_u64(seed, i, 0, 1) % 5 for i in range(len(x))], np.int32)
    return np.asarray(x, np.int32), np.asarray(y, np.int32), vm


def main():
    assert O.have_reference(), "oracle/_ref is not built: run `make -C oracle` with /root/reference present"
    for name, cells, boundary, potential, g, n, v, steps, seed in scenarios():
        field = O.ref_static_field(cells, boundary)
        x0, y0, vm = roster(cells, n, v, seed)
        st = O.RefState(cells, field, x0, y0, vm, boundary=boundary, potential=potential, drive_gradient=g)
        des, pos, alive, order, exited, hashes, disp = [], [], [], [], [], [], []
        for s in range(steps):
            alive_ids = np.flatnonzero(st.agents()[2])
            order.append(alive_ids[O.movement_order(len(alive_ids), seed, s)] if len(alive_ids) else alive_ids)
            st.plan(K_S, seed)
            dx, dy = st.desired()
            des.append(np.stack([dx, dy]))
            ex, d = st.move(seed)
            disp.append(d)
            st.step = st.step + 1
            x, y, a = st.agents()
            pos.append(np.stack([x, y]))
            alive.append(a.copy())
            exited.append(np.asarray(ex, np.int64))
            hashes.append(st.hash())
        ex_flat = np.concatenate(exited) if exited else np.zeros(0, np.int64)
        ex_off = np.cumsum([0] + [len(e) for e in exited])
        ord_flat = np.concatenate(order)
        ord_off = np.cumsum([0] + [len(o) for o in order])
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"), cells=cells, boundary=boundary, potential=potential,
            drive_gradient=g, k_s=K_S, seed=seed, field=field, x0=x0, y0=y0, v_max=vm,
            desired=np.array(des, np.int32), pos=np.array(pos, np.int32), alive=np.array(alive, np.uint8),
            exited=ex_flat, exited_off=ex_off, order=ord_flat, order_off=ord_off,
            state_hash=np.array(hashes, np.uint64), displacement=np.array(disp, np.int64))
        print(f"{name}: {cells.shape[1]}x{cells.shape[0]}, {len(x0)} agents, {steps} steps, "
              f"{len(ex_flat)} exits, final alive {int(alive[-1].sum())}")


if __name__ == "__main__":
    main()
