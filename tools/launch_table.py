"""Dev tool: per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, agg, cnt = None, collections.OrderedDict(), collections.Counter()
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h is None or len(r) < len(h):
        continue
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0].replace("void ", "")[:64]
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    us = v / 1000 if u == "nsecond" else v if u == "usecond" else v * 1000 if u == "msecond" else v * 1e6
    agg[k] = agg.get(k, 0) + us
    cnt[k] += 1
tot = sum(agg.values())
print(f"total {tot / 1000:.3f} ms over {sum(cnt.values())} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
    print(f"  {k:64s} n={cnt[k]:5d} {v / 1000:8.3f} ms")
