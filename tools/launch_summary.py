"""Dev tool: per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list.
usage: python tools/launch_summary.py launches.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
h, agg = None, collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            v *= {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(d.get("Metric Unit", ""), 1.0)
            agg[d["Kernel Name"][:70]][0] += 1
            agg[d["Kernel Name"][:70]][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"  {v[1] / 1e6:9.3f} ms {100 * v[1] / tot:5.1f}% x{v[0]:5d}  {k}")
