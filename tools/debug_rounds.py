"""Per-round timeline of the motion phase's grid rounds at a late step of a config.
python tools/debug_rounds.py --config plaza --warm 380"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp  # noqa: E402
from paper_0911_2900_b200 import scenarios  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="plaza")
ap.add_argument("--warm", type=int, default=380)
args = ap.parse_args()
wl = scenarios.build(args.config)
st = fp.SimState(wl.grid, None, wl.roster)
if wl.potential:
    st.set_potential(wl.potential, wl.drive_gradient)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=args.warm)
fp.run(st, p)
p.steps = 1
fp.run(st, p)
c = st.counters()
lib = fp.library()
t, n, ck, cm, pm = (np.zeros(64, np.int64) for _ in range(5))
ptr = lambda v: v.ctypes.data_as(C.c_void_p)  # noqa: E731
k = lib.fp_debug_rounds(st._ctx, ptr(t), ptr(n), ptr(ck), ptr(cm), ptr(pm), 64)
lib.fp_debug_rounds(st._ctx, ptr(t), ptr(n), ptr(ck), ptr(cm), ptr(pm), 64)
print("largest bucket (entries in one cell, reported when > 12):", cm[63])
print("seed_ns", c["motion_seed_ns"], "prep_ns", c["motion_prep_ns"], "grid_ns", c["motion_grid_ns"],
      "tail_ns", c["motion_tail_ns"], "contended", c["motion_contended"])
for r in range(k):
    dt = t[r + 1] - t[r] if r + 1 < k else 0
    print(f"round {r:3d} t={t[r]/1e3:8.1f} us pending={n[r]:8d} dur={dt/1e3:7.1f} us checks={ck[r]:7d} "
          f"pass2_max={cm[r]/1.965e3:7.1f} us pass1_max={pm[r]/1.965e3:7.1f} us")
