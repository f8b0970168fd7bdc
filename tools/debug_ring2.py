import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_0911_2900_b200 import fastped as fp, scenarios
import oracle as O
wl = scenarios.ring()
ro = wl.roster
st = fp.SimState(wl.grid, None, ro); st.set_potential(fp.DRIVE_X, wl.drive_gradient)
orc = O.State(wl.grid.cells, np.zeros(wl.grid.cells.shape), ro.x, ro.y, ro.v_max, boundary=1, potential=1, drive_gradient=wl.drive_gradient)
for s in range(10):
    fp.plan_phase(st, fp.SimParams(seed=1)); orc.plan(1.2, 1)
    dx, dy = st.desired()
    dm = np.nonzero((dx != orc.dx) | (dy != orc.dy))[0]
    x0, y0, _ = st.agents()
    mv = fp.move_phase(st, fp.SimParams(seed=1)); ex, disp = orc.move(1)
    st.step = st.step + 1; orc.step = orc.step + 1
    x, y, a = st.agents()
    bad = np.nonzero((x != orc.x) | (y != orc.y))[0]
    print("step", s, "desired mismatch", len(dm), "moved mismatch", len(bad))
    if len(dm):
        i = dm[0]
        print("   agent", i, "pos", x0[i], y0[i], "dev", dx[i], dy[i], "orc", orc.dx[i], orc.dy[i], "tile", x0[i] // 56, y0[i] // 16)
        break
    if len(bad): break
