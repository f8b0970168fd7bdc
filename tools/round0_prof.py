"""Round-0 breakdown of the motion rounds (build with -DFP_ROUND_PROF)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp, scenarios  # noqa: E402

L = fp.library()
L.fp_debug_rounds.argtypes = [C.c_void_p] + [C.c_void_p] * 5 + [C.c_int]
wl = scenarios.build("plaza")
st = fp.SimState(wl.grid, None, wl.roster)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
for s in range(201):
    fp.step(st, p)
    if s in (1, 200):
        arr = [np.zeros(64, np.int64) for _ in range(5)]
        L.fp_debug_rounds(st._ctx, *[a.ctypes.data for a in arr], 64)
        q = arr[4]
        print(f"step {s}: round0 checks {arr[2][0]} chk_clk {arr[3][0]} pass2 max {q[40]} cyc; local iters max cyc "
              f"{q[41:44].tolist()}; checks/iter {q[44:47].tolist()}; pending at iter {q[48:51].tolist()}")
