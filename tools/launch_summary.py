"""Aggregates an ncu --metrics gpu__time_duration.sum --csv launch list per kernel (ms, count)."""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
agg = collections.OrderedDict()
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0][:70]
    v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1e-6)
    agg.setdefault(k, [0.0, 0])
    agg[k][0] += v
    agg[k][1] += 1
tot = sum(a[0] for a in agg.values())
for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{t:9.3f} ms {c:4d}  {100 * t / tot:5.1f}%  {k}")
print(f"{tot:9.3f} ms total")
