"""Plan-kernel profile counters (FP_PLAN_PROF build via FASTPED_B200_LIB): producer ref waits,
consumer publish waits, per-warp-iteration cycles and lane occupancy, on plaza start/end."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_0911_2900_b200 import fastped as fp, scenarios  # noqa: E402

L = fp.library()
L.fp_debug_plan_prof.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
cfg = sys.argv[1] if len(sys.argv) > 1 else "plaza"
wl = scenarios.build(cfg)
st = fp.SimState(wl.grid, None, wl.roster)
if wl.potential:
    st.set_potential(wl.potential, wl.drive_gradient)


def prof(tag):
    ms = st.time_plan_kernel(wl.k_s, wl.seed, 1)
    o = np.zeros(8, np.int64)
    L.fp_debug_plan_prof(st._ctx, o.ctypes.data, 8)
    sms = 148
    print(f"{tag}: TMA issue {o[7]/max(o[1],1):.0f} cyc/load; longest consumer warp {o[2]/1.965e3:.0f} us; "
          f"publish waits {o[3]/1.965e3/148/12:.0f} us per warp")
    print(f"{tag}: {ms*1e3:.1f} us | producer ref-wait {o[0]/max(o[1],1):.0f} cyc x {o[1]} loads "
          f"({o[0]/sms/1.965e3:.1f} us/SM) | publish-wait {o[2]/max(o[3],1):.0f} cyc x {o[3]} "
          f"| warp-iter {o[4]/max(o[5],1):.0f} cyc x {o[5]}, {o[6]/max(o[5],1):.1f} agents/iter", flush=True)


prof("start")
fp.run(st, fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=int(sys.argv[2]) if len(sys.argv) > 2 else 396))
prof("end")
