import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_0911_2900_b200 import fastped as fp, scenarios
import oracle as O
wl = scenarios.ring()
ro = wl.roster
st = fp.SimState(wl.grid, None, ro); st.set_potential(fp.DRIVE_X, wl.drive_gradient)
orc = O.State(wl.grid.cells, np.zeros(wl.grid.cells.shape), ro.x, ro.y, ro.v_max, boundary=1, potential=1, drive_gradient=wl.drive_gradient)
fp.plan_phase(st, fp.SimParams(seed=1)); orc.plan(1.2, 1)
dx, dy = st.desired()
print("desired mismatch", int(((dx != orc.dx) | (dy != orc.dy)).sum()))
mv = fp.move_phase(st, fp.SimParams(seed=1)); ex, disp = orc.move(1)
x, y, a = st.agents()
bad = np.nonzero((x != orc.x) | (y != orc.y))[0]
print("moved mismatch", len(bad), "disp", mv.displacement_cells, disp, "counters", st.counters())
order = O.movement_order(len(ro.x), 1, 0)
rank = np.empty(len(order), np.int64); rank[order] = np.arange(len(order))
for i in bad[:8]:
    print(" agent", i, "rank", rank[i], "start", ro.x[i], ro.y[i], "desired", dx[i], dy[i], "dev", x[i], y[i], "orc", orc.x[i], orc.y[i])
