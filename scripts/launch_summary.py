"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list.
    python scripts/launch_summary.py launches.csv > summary.txt"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and "Kernel Name" in r)
h = rows[hi]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
cnt, tot = collections.Counter(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0]
        cnt[name] += 1
        tot[name] += float(r[vi].replace(",", ""))
print("kernel | launches | avg gpu__time_duration (ns) | total (ns)")
for k, t in tot.most_common():
    print(f"{k} | {cnt[k]} | {t / cnt[k]:.0f} | {t:.0f}")
