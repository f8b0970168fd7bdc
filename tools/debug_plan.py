"""Per-fetch timeline of one plan CTA (DEBUG build only): issue, TMA ready, last agent done."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp  # noqa: E402
from paper_0911_2900_b200 import scenarios  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 0
wl = scenarios.build("plaza")
st = fp.SimState(wl.grid, None, wl.roster)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=max(warm, 1))
fp.run(st, p)
lib = fp.library()
buf = np.zeros(1024, np.uint64)
buf[256:512] = np.iinfo(np.uint64).max
# reset: write via a dummy copy to the symbol is not exposed; rely on a fresh process per call
ms = st.time_plan_kernel(wl.k_s, wl.seed, 1)
lib.fp_debug_plan(buf.ctypes.data_as(C.c_void_p))
iss, rdy, done, cnt = buf[:256].astype(np.int64), buf[256:512], buf[512:768].astype(np.int64), buf[768:].astype(np.int64)
t0 = iss[0]
print("plan kernel %.3f ms" % ms)
for i in range(256):
    if iss[i] == 0:
        break
    r = int(rdy[i]) - t0
    print(f"fetch {i:3d} issue {(iss[i]-t0)/1e3:7.2f} us ready {r/1e3:7.2f} done {(done[i]-t0)/1e3:7.2f} agents {cnt[i]:4d}")
