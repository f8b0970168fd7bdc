"""Race probe for the motion: repeated full plaza runs (fp_run, and step by step) must all end
on the same state hash."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp, scenarios  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "plaza"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 396
wl = scenarios.build(cfg)
hs = []
for i in range(reps):
    st = fp.SimState(wl.grid, None, wl.roster)
    if wl.potential:
        st.set_potential(wl.potential, wl.drive_gradient)
    fp.run(st, fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=steps))
    hs.append(fp.state_hash(st))
    print(f"rep {i}: hash {hs[-1]}", flush=True)
    st.close() if hasattr(st, "close") else None
print("OK" if len(set(hs)) == 1 else "MISMATCH", len(set(hs)))
