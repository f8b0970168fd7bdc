"""Plan-kernel launch time on a config's start state only (A/B of library variants via
FASTPED_B200_LIB): python tools/plan_start_time.py [config] [label]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp, scenarios  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "plaza"
label = sys.argv[2] if len(sys.argv) > 2 else os.environ.get("FASTPED_B200_LIB", "default")
wl = scenarios.build(cfg)
st = fp.SimState(wl.grid, None, wl.roster)
if wl.potential:
    st.set_potential(wl.potential, wl.drive_gradient)
st.time_plan_kernel(wl.k_s, wl.seed, 3)
t = st.time_plan_kernel(wl.k_s, wl.seed, 20)
print(f"{label} {cfg}: plan start {t*1e3:.1f} us", flush=True)
