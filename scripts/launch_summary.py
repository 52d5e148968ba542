"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    v *= scale.get(d["Metric Unit"], 1.0)
    name = d["Kernel Name"].split("(")[0][:70]
    agg.setdefault(name, []).append(v)
tot = sum(sum(v) for v in agg.values())
print(f"{'total us':>10} {'n':>4} {'avg us':>9} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):10.1f} {len(v):4d} {sum(v)/len(v):9.1f} {100*sum(v)/tot:5.1f}%  {k}")
