"""A small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): the
production step (plan stream kernel, exact path, order, motion rounds incl. the bucket rounds
and the shared-memory tail) on a crowded room, plus two virtual strips, checked against the
single-context run."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_0911_2900_b200 import fastped as fp  # noqa: E402

W, H = 300, 120
cells = np.zeros((H, W), np.uint8)
cells[0, :] = cells[-1, :] = 1
cells[:, 0] = cells[:, -1] = 1
cells[-1, 140:146] = 2
cells[40:80, 100] = 1
grid = fp.Grid(cells)
x, y = O.spawn_agents(cells, 9000, 3)
ro = fp.Roster(np.asarray(x, np.int32), np.asarray(y, np.int32), np.full(len(x), 4, np.int32),
               np.ones(len(x), np.uint8))
st = fp.SimState(grid, None, ro)
ss = fp.StripSet(grid, None, ro, 2)
p = fp.SimParams(k_s=1.2, seed=5, steps=1)
for s in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    a = fp.step(st, p)
    b = ss.step(p)
    assert (a.alive, a.exited, a.displacement_cells) == (b.alive, b.exited, b.displacement_cells)
assert ss.state_hash() == fp.state_hash(st)
print("ok", st.counters()["motion_contended"], fp.state_hash(st))
