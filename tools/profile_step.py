"""Short driver for ncu captures: builds a config, warms up, then runs the chosen stage.

  python tools/profile_step.py --config plaza --mode plan   # plan kernel launches only
  python tools/profile_step.py --config plaza --mode run    # full steps (graph replays)
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0911_2900_b200 import fastped as fp  # noqa: E402
from paper_0911_2900_b200 import scenarios  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="plaza")
ap.add_argument("--mode", default="plan", choices=["plan", "run"])
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()
wl = scenarios.build(args.config)
st = fp.SimState(wl.grid, None, wl.roster)
if wl.potential:
    st.set_potential(wl.potential, wl.drive_gradient)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=args.steps)
fp.run(st, p)  # warm: plane, graphs, reservations
if args.mode == "plan":
    print("plan ms", st.time_plan_kernel(wl.k_s, wl.seed, args.steps))
else:
    r = fp.run(st, p)
    print("run", r)
print("counters", st.counters())
