"""DESIGN.md section-5 table from bench lines: python tools/results_table.py DIR (bench_*.json)."""
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "profiles"
pre = sys.argv[2] if len(sys.argv) > 2 else "r02_bench_"
rows = [("plaza", "plaza (config 4), 396 steps"), ("plaza20", "plaza, first 20 steps"),
        ("room_v1", "room (config 2) v=1"), ("room_v2", "room v=2"), ("room_v3", "room v=3"),
        ("room_v4", "room v=4"), ("room_v5", "room v=5"), ("ring", "ring (config 3), FD on"),
        ("corridor", "corridor (config 1)"), ("obstacles", "obstacles (config 5), first 20 steps")]
print("| Config (1×B200) | agent-updates/s (device) | ms/step | e2e (C ABI, host buffers) | reference CPU "
      "(16 cores) | device ÷ CPU | plan launch start / end | plan-kernel roofline start / end |")
print("|---|---|---|---|---|---|---|---|")
for k, name in rows:
    p = os.path.join(d, pre + k + ".json")
    if not os.path.exists(p):
        continue
    try:
        b = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception:
        continue
    cpu = (b.get("cpu_baseline") or {}).get("value")
    e2e = (b.get("e2e") or {}).get("value")
    rf = b.get("roofline") or {}
    stt = rf.get("states", {})
    s, e = stt.get("start", {}), stt.get("end", {})
    ratio = f"{b['value'] / cpu:.0f}×" if cpu else "-"
    print(f"| {name} | {b['value']:.3g} | {b['ms_per_step']:.3f} | {e2e:.3g} | {cpu:.3g} | {ratio} | "
          f"{s.get('plan_ms', 0) * 1e3:.0f} / {e.get('plan_ms', 0) * 1e3:.0f} µs | "
          f"{s.get('frac', 0):.2f} / {e.get('frac', 0):.2f} |")
