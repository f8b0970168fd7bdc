"""Per-CTA start/end of one plan launch (DEBUG build): load balance of the tile deal."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp  # noqa: E402
from paper_0911_2900_b200 import scenarios  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 1
wl = scenarios.build("plaza")
st = fp.SimState(wl.grid, None, wl.roster)
fp.run(st, fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=max(warm, 1)))
ms = st.time_plan_kernel(wl.k_s, wl.seed, 1)
buf = np.zeros(768, np.uint64)
fp.library().fp_debug_plan_cta(buf.ctypes.data_as(C.c_void_p))
g = 148
st_, en, nf = buf[:g].astype(np.int64), buf[256:256 + g].astype(np.int64), buf[512:512 + g]
t0 = st_.min()
dur = (en - st_) / 1e3
print("plan kernel %.3f ms; CTA start spread %.1f us; CTA durations us: min %.1f median %.1f max %.1f; "
      "end spread %.1f us" % (ms, (st_.max() - t0) / 1e3, dur.min(), np.median(dur), dur.max(), (en.max() - en.min()) / 1e3))
order = np.argsort(-dur)[:8]
print("slowest CTAs:", [(int(b), round(float(dur[b]), 1), int(nf[b])) for b in order])
print("fetches per CTA: min %d median %d max %d" % (nf.min(), np.median(nf), nf.max()))
