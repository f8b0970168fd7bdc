"""Setup cost of compute_static_field (field.cu, world.hpp:220-266) at the full-size geometries:
wall clock of fp_static_field (host cells in, fp64 field out), second call of each; with `cpu`
also the compiled reference's Dijkstra on the plaza for scale (checker-side, oracle/_ref)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import fastped as fp, scenarios  # noqa: E402

for cfg, kw in (("room", {}), ("plaza", {"n": 1000}), ("obstacles", {"n": 1000})):
    wl = scenarios.build(cfg, **kw)
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        f = fp.compute_static_field(wl.grid)
        ts.append(time.perf_counter() - t0)
    print(f"{cfg}: {wl.grid.width}x{wl.grid.height} = {wl.grid.width * wl.grid.height / 1e6:.0f}M cells, "
          f"device field {ts[1] * 1e3:.0f} ms (first call {ts[0] * 1e3:.0f} ms)", flush=True)
    if cfg == "plaza" and "cpu" in sys.argv[1:]:
        import oracle as O  # noqa: E402
        t0 = time.perf_counter()
        g = O.ref_static_field(wl.grid.cells, 0)
        print(f"  reference Dijkstra on one host core: {(time.perf_counter() - t0) * 1e3:.0f} ms; "
              f"bitwise equal: {g.tobytes() == f.tobytes()}", flush=True)
