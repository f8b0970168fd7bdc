"""Motion prep sub-phase times (build with -DFP_PREP_PROF; FASTPED_B200_LIB=that library)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp, scenarios  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "plaza"
marks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 200, 395]
L = fp.library()
L.fp_debug_rounds.argtypes = [C.c_void_p] + [C.c_void_p] * 5 + [C.c_int]
wl = scenarios.build(cfg)
st = fp.SimState(wl.grid, None, wl.roster)
if wl.potential:
    st.set_potential(wl.potential, wl.drive_gradient)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
names = ["p2_number", "bk_count", "scan_count", "scan_base", "bk_place", "bk_sort", "bk_sort_long"]
for s in range(max(marks) + 1):
    fp.step(st, p)
    if s in marks:
        arr = [np.zeros(64, np.int64) for _ in range(5)]
        L.fp_debug_rounds(st._ctx, *[a.ctypes.data for a in arr], 64)
        t = arr[4][39:47]
        c = st.counters()
        print(f"step {s}: contended {c['motion_contended']}: " +
              ", ".join(f"{n} {(t[i + 1] - t[i]) / 1e3:.1f}" for i, n in enumerate(names)) + " us")
