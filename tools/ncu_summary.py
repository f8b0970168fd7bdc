"""Summarise an ncu report: key metrics, stall reasons, top stalled SASS lines.
usage: python tools/ncu_summary.py report.ncu-rep [n_top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 15
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, vals = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]
for v in vals:
    print("kernel:", v[h.index("Kernel Name")][:60] if "Kernel Name" in h else "")
    for w in want:
        if w in h:
            print(f"  {w} = {v[h.index(w)]} {units[h.index(w)]}")
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                st.append((float(v[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in st) or 1
    print("  stalls:", ", ".join(f"{n} {100*s/tot:.0f}%" for s, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
if len(srows) > 2:
    sh = srows[1]
    data = srows[2:]
    iS = sh.index("Warp Stall Sampling (All Samples)")
    iE = sh.index("Instructions Executed")
    iA = sh.index("Avg. Threads Executed")
    print("  top stalled SASS (samples, executed, avg threads, instr):")
    for k, r in sorted(enumerate(data), key=lambda t: -int(t[1][iS] or 0))[:ntop]:
        print(f"   #{k:5d} {r[iS]:>6} {r[iE]:>9} {r[iA]:>3}  {r[1][:70]}")
# per CUDA source line: samples attributed to the SASS under each line (cuda,sass view)
mix = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, fname, line, hdr = {}, "", "", None
for r in csv.reader(io.StringIO(mix)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:
        line = (fname, int(r[0]), r[1].strip()[:60])
    elif r[4] not in ("-", ""):
        agg[line] = agg.get(line, 0) + int(r[4])
tot = sum(agg.values()) or 1
print("  top source lines (stall samples %):")
for (f, ln, txt), s in sorted(agg.items(), key=lambda t: -t[1])[:ntop]:
    print(f"   {100*s/tot:5.1f}%  {f}:{ln}  {txt}")
