"""Motion-phase breakdown (device globaltimer counters of fp_counters) along a plaza run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp, scenarios  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "plaza"
kw = {"n": int(sys.argv[2])} if len(sys.argv) > 2 else {}  # e.g. plaza 32768000: a capacity probe's roster
wl = scenarios.build(cfg, **kw)
st = fp.SimState(wl.grid, None, wl.roster)
if wl.potential:
    st.set_potential(wl.potential, wl.drive_gradient)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
marks = {1, 10, 50, 100, 150, 200, 250, 300, 350, 395}
tot = 0.0
for s in range(396):
    t0 = __import__("time").perf_counter()
    fp.step(st, p)
    dt = __import__("time").perf_counter() - t0
    if s in marks:
        print(f"  step wall {dt * 1e3:.2f} ms", end=" ")
        c = st.counters()
        us = lambda k: c[k] / 1e3  # noqa: E731
        print(f"step {s:3d}: alive {st.alive} contended {c['motion_contended']:7d} | mark {us('motion_mark_ns'):6.1f} "
              f"seed {us('motion_seed_ns'):6.1f} prep {us('motion_prep_ns'):6.1f} grid {us('motion_grid_ns'):6.1f} "
              f"({c['motion_grid_rounds']} rounds) tail {us('motion_tail_ns'):6.1f} us", flush=True)
