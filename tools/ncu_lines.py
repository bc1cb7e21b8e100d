"""Dev tool: per-source-line samples, instructions and dominant stall reasons from an ncu
source-page CSV (--print-source cuda,sass)."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None; cur = None; fname = ""; src = {}
agg = defaultdict(lambda: defaultdict(float))
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; continue
    if r[0] != "": cur = (fname, int(r[0])); src[cur] = r[1]; continue
    if hdr is None: continue
    for i, h in enumerate(hdr):
        if i >= len(r): break
        if h.startswith("stall_") and "Not Issued" not in h or h in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
            try: agg[cur][h] += float(r[i] or 0)
            except ValueError: pass
S = "Warp Stall Sampling (All Samples)"
ts = sum(v[S] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][S])[:top]:
    st = sorted(((h[6:], x) for h, x in v.items() if h.startswith("stall_")), key=lambda y: -y[1])[:3]
    sts = " ".join(f"{h}:{x/max(v[S],1)*100:.0f}%" for h, x in st)
    print(f"{k[0][:12]:12s}{k[1]:5d} {v[S]/ts*100:5.1f}% inst {v['Instructions Executed']:10.0f} [{sts}] | {src[k][:70]}")
