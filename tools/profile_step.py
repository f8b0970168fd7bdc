"""Short driver for ncu captures and motion counters: builds a config, advances it, then runs
the chosen stage and prints the engine counters of the last motion phase.

  python tools/profile_step.py --config plaza --mode plan            # plan kernel launches only
  python tools/profile_step.py --config plaza --mode run             # full steps (graph replays)
  python tools/profile_step.py --config plaza --warm 300 --mode run  # from step 300
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
ap.add_argument("--warm", type=int, default=None, help="steps to advance first (default: --steps)")
ap.add_argument("--each", action="store_true", help="print counters after every step")
args = ap.parse_args()
wl = scenarios.build(args.config)
st = fp.SimState(wl.grid, None, wl.roster)
if wl.potential:
    st.set_potential(wl.potential, wl.drive_gradient)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=args.warm if args.warm is not None else args.steps)
if p.steps > 0:
    fp.run(st, p)  # warm: plane, graphs, reservations; advances the state
p.steps = args.steps
keys = ["motion_seed_ns", "motion_mark_ns", "motion_grid_ns", "motion_prep_ns", "motion_tail_ns",
        "motion_grid_rounds", "motion_contended"]
if args.mode == "plan":
    print("plan ms", st.time_plan_kernel(wl.k_s, wl.seed, args.steps))
elif args.each:
    p.steps = 1
    for _ in range(args.steps):
        r = fp.run(st, p)
        c = st.counters()
        print(f"step {st.step} plan {r.plan_time_s*1e3:.3f} ms move {r.move_time_s*1e3:.3f} ms alive {r.alive}",
              {k: c[k] for k in keys})
else:
    r = fp.run(st, p)
    print("run", r)
print("counters", st.counters())
