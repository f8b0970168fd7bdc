"""Regenerates the FULL-SIZE trajectory fixtures (tests/golden/full_*.npz) by running the
REFERENCE engine itself -- the unmodified headers compiled into oracle/_ref by oracle/Makefile --
on BASELINE.json's configurations at their full sizes:

    room1000 v = 1..5   40,000 agents        396 steps
    corridor 250x50      2,000 agents        396 steps
    ring 4000x200      182,000 agents        396 steps (DriveX, g = 1)
    plaza 20000x5000 1,000,000 agents        396 steps
    obstacles 40000x10000 10,000,000 agents  100 steps (mixed v_max 2..5; FASTPED_OBSTACLES_STEPS)

    python tests/golden/make_fullsize.py [name ...]     # ~30 min on 8 cores (obstacles: ~12 s per step)

Geometry and roster come from oracle/configs.py (the checker-side generators; the roster is the
reference's own spawn_agents), the static field from the reference's compute_static_field,
plan_phase / move_phase from the reference.  Per step the fixture keeps: state_hash after the
step (state.hpp:80-95), the alive count, the displacement (MoveOutcome::displacement_cells), the
exited ids in processing order, and a digest of the desired cells of the agents alive entering
the step (oracle.configs.desired_digest).  The initial roster and the cells are pinned by
sha256 so the GPU test (tests/test_fullsize_golden.py) can rebuild the same state from the
product's generators without /root/reference.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import oracle.configs as OC  # noqa: E402

CASES = {
    "room_v1": ("room", dict(v=1), 396),
    "room_v2": ("room", dict(v=2), 396),
    "room_v3": ("room", dict(v=3), 396),
    "room_v4": ("room", dict(v=4), 396),
    "room_v5": ("room", dict(v=5), 396),
    "corridor": ("corridor", {}, 396),
    "ring": ("ring", {}, 396),
    "plaza": ("plaza", {}, 396),
    "obstacles": ("obstacles", {}, int(os.environ.get("FASTPED_OBSTACLES_STEPS", "100"))),
}


def make(name: str, cores: int) -> None:
    cfg_name, kw, steps = CASES[name]
    t0 = time.time()
    cfg = OC.build(cfg_name, **kw)
    st = O.RefState(cfg.cells, None, cfg.x, cfg.y, cfg.v, boundary=cfg.boundary, potential=cfg.potential,
                    drive_gradient=cfg.drive_gradient)
    t1 = time.time()
    hashes, alive, disp, ex_all, ex_off, dd = [], [], [], [], [0], []
    h0 = st.hash()
    for s in range(steps):
        a_before = st.agents()[2].astype(bool)
        st.plan(cfg.k_s, cfg.seed, cores)
        dx, dy = st.desired()
        dd.append(OC.desired_digest(dx, dy, a_before))
        ex, d = st.move(cfg.seed)
        st.step = st.step + 1
        hashes.append(st.hash())
        alive.append(st.alive_count)
        disp.append(d)
        ex_all.append(np.asarray(ex, np.uint32))
        ex_off.append(ex_off[-1] + len(ex))
        if cfg.n >= 1_000_000 and s % 10 == 9:
            print(f"  {name}: step {s + 1}/{steps}, {time.time() - t1:.0f} s", file=sys.stderr, flush=True)
    t2 = time.time()
    np.savez_compressed(
        os.path.join(HERE, f"full_{name}.npz"), config=cfg_name, kwargs=repr(kw), steps=steps, k_s=cfg.k_s,
        seed=cfg.seed, cells_sha256=OC.cells_digest(cfg.cells), roster_sha256=OC.roster_digest(cfg.x, cfg.y, cfg.v),
        hash0=np.uint64(h0), state_hash=np.array(hashes, np.uint64), alive=np.array(alive, np.int64),
        displacement=np.array(disp, np.int64), desired_digest=np.array(dd, np.uint64),
        exited=np.concatenate(ex_all) if ex_all else np.zeros(0, np.uint32), exited_off=np.array(ex_off, np.int64))
    print(f"{name}: {cfg.cells.shape[1]}x{cfg.cells.shape[0]}, {cfg.n} agents, {steps} steps, "
          f"{ex_off[-1]} exits, final alive {alive[-1]}; setup {t1 - t0:.1f} s, steps {t2 - t1:.1f} s", flush=True)


def main():
    assert O.have_reference(), "oracle/_ref is not built: run `make -C oracle` with /root/reference present"
    names = sys.argv[1:] or list(CASES)
    cores = O.physical_core_count()
    for n in names:
        make(n, cores)


if __name__ == "__main__":
    main()
