"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
total time per kernel name (us), launches, share."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    u = d.get("Metric Unit", "")
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
    k = d["Kernel Name"][:90]
    agg.setdefault(k, [0, 0.0])
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v:12.1f} us {n:5d}  {100 * v / tot:5.1f}%  {k}")
print(f"{tot:12.1f} us total")
