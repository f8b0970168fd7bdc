"""Where the end-to-end (host-buffer) step time goes over a full run from step 0:
fp_update_agents, fp_step, fp_get_agents (wall clock per call, averaged)."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp  # noqa: E402
from paper_0911_2900_b200 import scenarios  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="plaza")
ap.add_argument("--steps", type=int, default=396)
args = ap.parse_args()
wl = scenarios.build(args.config)
ro = wl.roster
st0 = fp.SimState(wl.grid, None, ro)
st = fp.SimState(wl.grid, st0.field(), ro)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
hx = torch.from_numpy(ro.x.copy()).pin_memory().numpy()
hy = torch.from_numpy(ro.y.copy()).pin_memory().numpy()
ha = torch.from_numpy(ro.alive.copy()).pin_memory().numpy()
fp.step(st0, p)  # warm the library / first capture on another context
t = np.zeros(3)
torch.cuda.synchronize()
T0 = time.perf_counter()
for s in range(args.steps):
    t0 = time.perf_counter()
    st.set_agents(hx, hy, ha)
    t1 = time.perf_counter()
    fp.step(st, p)
    t2 = time.perf_counter()
    st.agents(out=(hx, hy, ha))
    t3 = time.perf_counter()
    t += [t1 - t0, t2 - t1, t3 - t2]
T = time.perf_counter() - T0
print("%d steps: total %.3f ms/step  update_agents %.3f  step %.3f  get_agents %.3f" %
      ((args.steps, T / args.steps * 1e3) + tuple(t / args.steps * 1e3)))
st3 = fp.SimState(wl.grid, st0.field(), ro)
torch.cuda.synchronize()
T0 = time.perf_counter()
for s in range(args.steps):
    fp.step(st3, p)
torch.cuda.synchronize()
print("device-resident step() loop %.3f ms/step" % ((time.perf_counter() - T0) / args.steps * 1e3))
