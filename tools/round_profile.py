"""Per-round breakdown of the motion's grid rounds (fp_debug_rounds) at chosen plaza steps."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp, scenarios  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "plaza"
marks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 50, 200, 395]
L = fp.library()
L.fp_debug_rounds.argtypes = [C.c_void_p] + [C.c_void_p] * 5 + [C.c_int]
wl = scenarios.build(cfg)
st = fp.SimState(wl.grid, None, wl.roster)
if wl.potential:
    st.set_potential(wl.potential, wl.drive_gradient)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
for s in range(max(marks) + 1):
    fp.step(st, p)
    if s in marks:
        arr = [np.zeros(64, np.int64) for _ in range(5)]
        n = L.fp_debug_rounds(st._ctx, *[a.ctypes.data for a in arr], 64)
        c = st.counters()
        print(f"step {s}: contended {c['motion_contended']} prep_done->tail {c['motion_grid_ns']/1e3:.1f} us "
              f"largest bucket {arr[3][63]}")
        for r in range(n):
            print(f"  round {r:2d}: t {arr[0][r]/1e3:8.1f} us pending {arr[1][r]:8d} checks {arr[2][r]:8d} "
                  f"p1_clk {arr[4][r]:8d} chk_clk {arr[3][r]:8d}")
