"""Development tool: per-kernel totals and shares from an `ncu --metrics gpu__time_duration.sum --csv`
launch list.   usage: ncu_launches.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ix = {x: i for i, x in enumerate(h)}
scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    t = float(r[ix["Metric Value"]].replace(",", "")) * scale[r[ix["Metric Unit"]]]
    a = agg[r[ix["Kernel Name"]]]
    a[0] += 1
    a[1] += t
tot = sum(v[1] for v in agg.values())
print(f"| kernel | launches | total | share |\n|---|---:|---:|---:|")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k[:70]}` | {n} | {t:.6f} s | {100 * t / tot:.3f}% |")
