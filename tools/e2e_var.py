"""Variance probe of the e2e loop: per-phase averages and worst step, several repetitions."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp  # noqa: E402
from paper_0911_2900_b200 import scenarios  # noqa: E402

wl = scenarios.build("plaza")
ro = wl.roster
st0 = fp.SimState(wl.grid, None, ro)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
for rep in range(3):
    st = fp.SimState(wl.grid, st0.field(), ro)
    hx = torch.from_numpy(ro.x.copy()).pin_memory().numpy()
    hy = torch.from_numpy(ro.y.copy()).pin_memory().numpy()
    ha = torch.from_numpy(ro.alive.copy()).pin_memory().numpy()
    t = np.zeros((120, 3))
    for s in range(120):
        t0 = time.perf_counter()
        st.set_agents(hx, hy, ha)
        t1 = time.perf_counter()
        fp.step(st, p)
        t2 = time.perf_counter()
        st.agents(out=(hx, hy, ha))
        t3 = time.perf_counter()
        t[s] = [t1 - t0, t2 - t1, t3 - t2]
    m = t[1:].mean(0) * 1e3
    mx = t[1:].max(0) * 1e3
    print("rep %d: mean ms update %.3f step %.3f get %.3f | max %.3f %.3f %.3f | first step %.1f ms"
          % (rep, *m, *mx, t[0].sum() * 1e3))
    st.close()
