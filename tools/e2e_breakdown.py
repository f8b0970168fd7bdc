"""Where the end-to-end (host-buffer) step time goes: fp_update_agents, fp_step, fp_get_agents."""
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
st = fp.SimState(wl.grid, None, ro)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
hx = torch.from_numpy(ro.x.copy()).pin_memory().numpy()
hy = torch.from_numpy(ro.y.copy()).pin_memory().numpy()
ha = torch.from_numpy(ro.alive.copy()).pin_memory().numpy()
fp.step(st, p)
t = np.zeros(3)
for s in range(30):
    t0 = time.perf_counter()
    st.set_agents(hx, hy, ha)
    t1 = time.perf_counter()
    fp.step(st, p)
    t2 = time.perf_counter()
    st.agents(out=(hx, hy, ha))
    t3 = time.perf_counter()
    t += [t1 - t0, t2 - t1, t3 - t2]
print("per step ms: update_agents %.3f  step %.3f  get_agents %.3f" % tuple(t / 30 * 1e3))
x = np.empty(len(ro), np.int32)
t0 = time.perf_counter()
for _ in range(10):
    st.agents()
print("get_agents alone %.3f ms" % ((time.perf_counter() - t0) / 10 * 1e3))
