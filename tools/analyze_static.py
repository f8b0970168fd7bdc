"""How much of the motion phase's contention at a late plaza step comes from paths that run into
an agent that does not move this step (a 'static' blocker)?  Runs the engine to --warm, plans
one step, and analyses footprints on the host."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp  # noqa: E402
from paper_0911_2900_b200 import scenarios  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="plaza")
ap.add_argument("--warm", type=int, default=380)
args = ap.parse_args()
wl = scenarios.build(args.config)
st = fp.SimState(wl.grid, None, wl.roster)
p = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=args.warm)
fp.run(st, p)
fp.plan_phase(st, p)
x, y, a = st.agents()
dx, dy = st.desired()
al = a.astype(bool)
W, H = wl.grid.width, wl.grid.height
cells = wl.grid.cells
mover = al & ((dx != x) | (dy != y))
occ = np.zeros((H, W), bool)
occ[y[al], x[al]] = True
static = np.zeros((H, W), bool)
static[y[al & ~mover], x[al & ~mover]] = True


def path(x0, y0, x1, y1, v):
    out = []
    ddx, ddy = abs(x1 - x0), -abs(y1 - y0)
    sx, sy = (1 if x0 < x1 else -1), (1 if y0 < y1 else -1)
    err, cx, cy = ddx + ddy, x0, y0
    while (cx, cy) != (x1, y1) and len(out) < v:
        e2 = 2 * err
        if e2 >= ddy:
            err += ddy
            cx += sx
        if e2 <= ddx:
            err += ddx
            cy += sy
        out.append((cx, cy))
    return out


ids = np.flatnonzero(mover)
rng = np.random.default_rng(0)
sample = rng.choice(ids, size=min(200000, len(ids)), replace=False)
v = wl.roster.v_max
full, trunc, zero = 0, 0, 0
foot_full = np.zeros((H, W), np.int32)
foot_trunc = np.zeros((H, W), np.int32)
for i in sample:
    pth = path(x[i], y[i], dx[i], dy[i], int(v[i]))
    n = len(pth)
    k = n
    for j, (cx, cy) in enumerate(pth):
        if cells[cy, cx] == 1:
            k = j
            n = j
            break
        if static[cy, cx]:
            k = j
            break
    full += n
    trunc += k
    zero += (k == 0)
    foot_full[y[i], x[i]] += 1
    foot_trunc[y[i], x[i]] += 1
    for (cx, cy) in pth[:n]:
        foot_full[cy, cx] += 1
    for (cx, cy) in pth[:k]:
        foot_trunc[cy, cx] += 1
print(f"alive {al.sum()} movers {mover.sum()} sampled {len(sample)}")
print(f"mean path cells {full/len(sample):.2f}, truncated at static blockers {trunc/len(sample):.2f}, "
      f"movers blocked at the first cell by a static agent: {zero/len(sample):.3f}")
print("cells in >=2 sampled footprints: full", int((foot_full >= 2).sum()), "truncated", int((foot_trunc >= 2).sum()))
