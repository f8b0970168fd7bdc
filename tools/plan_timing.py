"""Plan-kernel launch time (CUDA events) on the plaza start state and after N steps, plus the
whole-step time; the quick A/B loop for plan.cu changes."""
import sys
import os
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp, scenarios  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "plaza"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 396
wl = scenarios.build(cfg)
st = fp.SimState(wl.grid, None, wl.roster)
if wl.potential:
    st.set_potential(wl.potential, wl.drive_gradient)
t0 = st.time_plan_kernel(wl.k_s, wl.seed, 20)
r = fp.run(st, fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=steps))
t1 = st.time_plan_kernel(wl.k_s, wl.seed, 20)
print(f"{cfg}: plan start {t0*1e3:.1f} us, end(step {steps}) {t1*1e3:.1f} us; run {r.wall_time_s/steps*1e3:.3f} ms/step "
      f"(plan {r.plan_time_s/steps*1e3:.3f}, move {r.move_time_s/steps*1e3:.3f}); hash {fp.state_hash(st)}", flush=True)
