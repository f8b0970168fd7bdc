"""Runs a BASELINE workload on the device for K steps and saves the roster (x, y, alive) to an
.npz -- input for offline tile/coverage analysis of the plan kernel's data layout."""
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp, scenarios  # noqa: E402

cfg, steps, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
wl = scenarios.build(cfg)
st = fp.SimState(wl.grid, None, wl.roster)
if wl.potential:
    st.set_potential(wl.potential, wl.drive_gradient)
if steps:
    fp.run(st, fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=steps))
x, y, a = st.agents()
np.savez_compressed(out, x=x, y=y, alive=a, v=wl.roster.v_max, step=steps)
print("saved", out, int(a.sum()))
