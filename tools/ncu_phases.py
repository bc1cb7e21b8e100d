"""Dev tool: attribute ncu source-page samples/instructions of the step kernel to phases."""
import csv, re, sys
from collections import defaultdict
path = sys.argv[1]
src_file = sys.argv[2] if len(sys.argv) > 2 else "/root/repo/paper_2311_04517_b200/csrc/step_kernel.cuh"
# phase boundaries from marker comments in the kernel source
marks = []
for i, line in enumerate(open(src_file), 1):
    m = re.search(r"// -{2,} ?(\w[\w ,:()'+/-]*)|// \((\d)\) (\w+)", line)
    if m:
        marks.append((i, (m.group(1) or ("seed-" + m.group(3))).strip()[:28]))
def phase(f, ln):
    if not f.endswith("step_kernel.cuh"):
        return "helpers:" + f[:20]
    name = "prologue"
    for i, nm in marks:
        if ln >= i: name = nm
    return name
rows = list(csv.reader(open(path)))
agg = defaultdict(lambda: [0.0, 0.0]); cur = None; fname = ""
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] in ("Line No", "Function Name"): continue
    if r[0] != "": cur = phase(fname, int(r[0])); continue
    try: s = float(r[4] or 0); i = float(r[7] or 0)
    except: continue
    agg[cur][0] += s; agg[cur][1] += i
ts = sum(v[0] for v in agg.values()); ti = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:40s} stall {v[0]/ts*100:5.1f}%  inst {v[1]/ti*100:5.1f}%")
