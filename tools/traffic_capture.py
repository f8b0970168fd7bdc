"""ncu DRAM bytes of the plan kernel on bench.py's start and end states -> profiles/plan_kernel_ncu.json
(the `traffic` of bench.py's roofline).  Run on the GPU box: python tools/traffic_capture.py plaza"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1] if len(sys.argv) > 1 else "plaza"
out_path = os.path.join(ROOT, "profiles", "plan_kernel_ncu.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
if not isinstance(res.get(cfg), dict) or "start" not in res.get(cfg, {}):
    res[cfg] = {}
skips = {"start": 1, "end": 397 if cfg != "obstacles" else 397}
for state, skip in skips.items():
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum", "--csv",
           "--clock-control", "none", "-k", "regex:plan_stream_kernel", "--launch-skip", str(skip), "--launch-count", "1",
           sys.executable, "bench.py", "--config", cfg, "--plan-state", state]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1800)
    rows = [r for r in csv.reader(io.StringIO(p.stdout)) if len(r) > 10]
    hdr = rows[0]
    vals = {r[hdr.index("Metric Name")]: (r[hdr.index("Metric Value")], r[hdr.index("Metric Unit")]) for r in rows[1:]}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(vals["dram__bytes_read.sum"][0].replace(",", "")) * scale[vals["dram__bytes_read.sum"][1]]
    wr = float(vals["dram__bytes_write.sum"][0].replace(",", "")) * scale[vals["dram__bytes_write.sum"][1]]
    t = vals["gpu__time_duration.sum"]
    res[cfg][state] = {"dram_bytes_per_launch": rd + wr, "dram_bytes_read": rd, "dram_bytes_write": wr,
                       "gpu_time_under_ncu": f"{t[0]} {t[1]}",
                       "capture": " ".join(cmd[:-4]).replace(sys.executable, "python") + f" ... --plan-state {state}"}
    print(cfg, state, res[cfg][state], flush=True)
json.dump(res, open(out_path, "w"), indent=1)
