"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if r[mi] != "gpu__time_duration.sum":
        continue
    agg[r[ki]][0] += 1
    agg[r[ki]][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
tot = sum(v[1] for v in agg.values())
print(f"# {sys.argv[2] if len(sys.argv) > 2 else ''}")
print("# launches  total_us  mean_us  share  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:8d} {t:11.1f} {t / n:8.2f} {100 * t / tot:6.2f}%  {k}")
