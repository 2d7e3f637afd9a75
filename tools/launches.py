"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0][:60]
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-6)
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} {c:6d} {t:9.3f} ms {100 * t / tot:5.1f}%  {1000 * t / c:8.1f} us/launch")
print(f"total {tot:.2f} ms")
