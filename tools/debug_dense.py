import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_0911_2900_b200 import fastped as fp, scenarios
import oracle as O
case = sys.argv[1]
if case == "ring":
    wl = scenarios.ring()
    g, ro = wl.grid, wl.roster
elif case == "dense":
    W = H = 120
    c = np.zeros((H, W), np.uint8); c[0,:]=c[-1,:]=c[:,0]=c[:,-1]=1; c[60, -1] = 2
    g = fp.Grid(c); ro = fp.spawn_agents(g, int(0.8 * (W-2)*(H-2)), 4, 3)
elif case == "half":
    W = H = 120
    c = np.zeros((H, W), np.uint8); c[0,:]=c[-1,:]=c[:,0]=c[:,-1]=1; c[60, -1] = 2
    g = fp.Grid(c); ro = fp.spawn_agents(g, int(0.3 * (W-2)*(H-2)), 4, 3)
st = fp.SimState(g, None, ro)
if case == "ring": st.set_potential(fp.DRIVE_X, 1.0)
try:
    fp.plan_phase(st, fp.SimParams(seed=1))
    print(case, "plan ok", st.counters())
except Exception as e:
    print(case, "plan FAILED", e)
