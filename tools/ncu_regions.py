"""Dev tool: attribute ncu per-instruction stall samples (source page, --print-source sass CSV) to
OUTERMOST kernel source lines (inlined helpers/lambdas charged to their call site), using
`nvdisasm -gi` of the same cubin. Usage: ncu_regions.py sass.csv disasm_gi.txt [regions]
regions: comma list of name:lo-hi line ranges of step_kernel.cuh."""
import csv, re, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iA, iS, iI = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stc = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
ins = [(int(r[iA], 16), float(r[iS] or 0), float(r[iI] or 0), {n: float(r[i] or 0) for i, n in stc})
       for r in rows[2:] if r and r[0].startswith("0x")]
base = ins[0][0]
loc = {}
group = []
for l in open(sys.argv[2]):
    if "//## File" in l:
        group.append(l)
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        if group:
            last = group[-1]
            mm = re.findall(r'"([^"]+)", line (\d+)', last)
            f, ln = mm[-1]
            cur = (f.split("/")[-1], int(ln))
            group = []
        loc[int(m.group(1), 16)] = cur
tot = sum(x[1] for x in ins)
agg = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
for a, s, n, st in ins:
    k = loc.get(a - base, ("?", 0))
    agg[k][0] += s; agg[k][1] += n
    for h, v in st.items(): agg[k][2][h] += v
def top(st, S):
    return " ".join(f"{h}:{v/max(S,1)*100:.0f}%" for h, v in sorted(st.items(), key=lambda x: -x[1])[:4])
if len(sys.argv) > 3:
    regs = []
    for part in sys.argv[3].split(","):
        nm, rg = part.split(":"); lo, hi = rg.split("-"); regs.append((nm, int(lo), int(hi)))
    ra = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
    for (f, ln), (s, n, st) in agg.items():
        nm = next((nm for nm, lo, hi in regs if f == "step_kernel.cuh" and lo <= ln <= hi), "other")
        ra[nm][0] += s; ra[nm][1] += n
        for h, v in st.items(): ra[nm][2][h] += v
    for nm, (s, n, st) in sorted(ra.items(), key=lambda x: -x[1][0]):
        print(f"{nm:14s} {s/tot*100:5.1f}%  inst {n:12.0f}  [{top(st, s)}]")
else:
    for k, (s, n, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:40]:
        print(f"{k[0][:16]:16s}{k[1]:5d} {s/tot*100:5.1f}% inst {n:12.0f}  [{top(st, s)}]")

# optional: instruction-level listing for one outer line: env LINE=<n>
import os
if os.environ.get("LINE"):
    want = int(os.environ["LINE"])
    text = {}
    for l in open(sys.argv[2]):
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m: text[int(m.group(1), 16)] = m.group(2).strip()
    for a, s, n, st in ins:
        off = a - base
        if loc.get(off, ("?", 0))[1] == want:
            print(f"{off:6x} {s:6.0f} {n:9.0f} {top(st, s):48s} {text.get(off, '')[:60]}")
