"""Plan-graph stage stamps (FP_STAGE_TIMING build via FASTPED_B200_LIB): per step, the globaltimer
of bucketing done, plan kernel done, exact path done, order select done, order done, join --
relative to the start of the plan graph; averaged over steps [a, b).
python tools/stage_timing.py [config] [a] [b]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_0911_2900_b200 import fastped as fp, scenarios  # noqa: E402

L = fp.library()
L.fp_debug_plan_prof.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
cfg = sys.argv[1] if len(sys.argv) > 1 else "plaza"
a = int(sys.argv[2]) if len(sys.argv) > 2 else 0
b = int(sys.argv[3]) if len(sys.argv) > 3 else 20
wl = scenarios.build(cfg)
st = fp.SimState(wl.grid, None, wl.roster)
if wl.potential:
    st.set_potential(wl.potential, wl.drive_gradient)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
if a > 0:
    p.steps = a
    fp.run(st, p)
    p.steps = 1
rows = []
for _ in range(b - a):
    fp.run(st, p)
    o = np.zeros(8, np.int64)
    L.fp_debug_plan_prof(st._ctx, o.ctypes.data, 8)
    rows.append((o - o[0]) / 1e3)
r = np.mean(rows, axis=0)
names = ["start", "bucketed", "plan kernel", "exact", "order start", "select", "order done", "joined"]
if os.environ.get("FP_STAGE_BUCKET"):
    names = ["start", "bucketed", "plan kernel", "exact", "counted", "scanned", "tile lists", "joined"]
print(cfg, f"steps {a}-{b}:", ", ".join(f"{n} {v:.1f}" for n, v in zip(names, r)), "us", flush=True)
