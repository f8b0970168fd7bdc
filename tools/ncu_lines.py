"""Per CUDA source line: warp instructions executed and stall samples of an ncu report
(--page source, cuda,sass view).  usage: python tools/ncu_lines.py report.ncu-rep [n_top] [file]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 40
only = sys.argv[3] if len(sys.argv) > 3 else None
mix = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, fname, line, hdr = {}, "", None, None
for r in csv.reader(io.StringIO(mix)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        iE = hdr.index("Instructions Executed")
        continue
    if hdr is None:
        continue
    if r[0]:
        line = (fname, int(r[0]), r[1].strip()[:70])
    if len(r) <= iE or r[iE] in ("-", ""):
        continue
    try:
        e = int(r[iE] or 0)
        st = int(r[iS] or 0)
    except (ValueError, IndexError):
        continue
    a = agg.setdefault(line, [0, 0])
    a[0] += e
    a[1] += st
tot_e = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot_e}, stall samples {tot_s}")
items = [(k, v) for k, v in agg.items() if k and (only is None or k[0] == only)]
for (f, ln, txt), (e, st) in sorted(items, key=lambda t: -t[1][0])[:ntop]:
    print(f"  {100*e/tot_e:5.1f}% inst {100*st/tot_s:5.1f}% stall  {f}:{ln}  {txt}")
