"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h, d = rows[i], rows[i + 1:]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
tot, cnt = collections.Counter(), collections.Counter()
for r in d:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        k = r[ki].split("(")[0].replace("void ", "")[:40]
        tot[k] += float(r[vi].replace(",", ""))
        cnt[k] += 1
skip = {k for k in tot if k.startswith(("field_", "plane_"))}  # setup, not the step
T = sum(v for k, v in tot.items() if k not in skip)
print(f"{'kernel':42s} {'launches':>8s} {'total us':>10s} {'share':>6s}")
for k, v in tot.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    share = "" if k in skip else f"{100 * v / T:5.1f}%"
    print(f"{k:42s} {cnt[k]:8d} {v / 1e3:10.1f} {share:>6s}")
print("step kernels total (us):", round(T / 1e3, 1))
