import sys, os
sys.path.insert(0, "/root/repo")
from paper_0911_2900_b200 import fastped as fp, scenarios
wl = scenarios.build("plaza")
st = fp.SimState(wl.grid, None, wl.roster)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
for s in range(201):
    fp.run(st, p)
    if s in (0, 1, 20, 100, 200):
        c = st.counters()
        print(s, {k: v for k, v in c.items() if k.startswith("motion") or k.startswith("plan")})
