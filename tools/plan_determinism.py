"""Race probe: the plan kernel replanned many times on fixed plaza states must give the same
desired cells every time (and the same as one fp_plan)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp, scenarios  # noqa: E402

wl = scenarios.build(sys.argv[1] if len(sys.argv) > 1 else "plaza")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
st = fp.SimState(wl.grid, None, wl.roster)
if wl.potential:
    st.set_potential(wl.potential, wl.drive_gradient)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
bad = 0
for stage in (0, 100, 200, 300, 396):
    while st.step < stage:
        fp.step(st, p)
    fp.plan_phase(st, p)
    rx, ry = (a.copy() for a in st.desired())
    for i in range(reps):
        st.time_plan_kernel(wl.k_s, wl.seed, 1)
        x, y = st.desired()
        d = int(np.count_nonzero((x != rx) | (y != ry)))
        if d:
            bad += 1
            idx = np.nonzero((x != rx) | (y != ry))[0][:5]
            print(f"step {stage} rep {i}: {d} desired cells differ, e.g. agents {idx.tolist()}", flush=True)
    print(f"step {stage}: {reps} replans checked", flush=True)
print("BAD" if bad else "OK", bad)
