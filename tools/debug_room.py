import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_0911_2900_b200 import fastped as fp, scenarios
import oracle as O
for v in (1, 4):
    wl = scenarios.room(v=v)
    ro = wl.roster
    st = fp.SimState(wl.grid, None, ro)
    orc = O.State(wl.grid.cells, O.static_field(wl.grid.cells), ro.x, ro.y, ro.v_max)
    for step in range(3):
        fp.plan_phase(st, fp.SimParams(seed=1))
        orc.plan(1.2, 1)
        dx, dy = st.desired()
        bad = np.nonzero((dx != orc.dx) | (dy != orc.dy))[0]
        print("v", v, "step", step, "mismatch", len(bad), "fallbacks", st.counters()["plan_fallbacks"])
        for i in bad[:5]:
            print("   agent", i, "pos", ro.x[i] if step == 0 else None, "dev", dx[i], dy[i], "orc", orc.dx[i], orc.dy[i])
        mv = fp.move_phase(st, fp.SimParams(seed=1)); st.step = st.step + 1
        orc.move(1); orc.step = orc.step + 1
