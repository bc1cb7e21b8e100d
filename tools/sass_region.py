"""Dev tool: SASS of one kernel instantiation whose OUTERMOST source line is in [lo, hi] of
step_kernel.cuh. Usage: sass_region.py <obj.o> <frag e.g. IfLi16E> <lo> <hi> [--count]"""
import re, subprocess, sys, tempfile, os
obj, frag, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cub)], capture_output=True, text=True).stdout
blk = next(b for b in re.split(r"\n\s*\.text\.", txt) if b.startswith("_ZN4hpcg18worker_step_kernel" + frag))
group, cur, inner, n = [], None, None, 0
from collections import Counter
ops = Counter()
for l in blk.split("\n"):
    if "//## File" in l:
        group.append(l); continue
    if re.search(r"/\*[0-9a-f]{4,}\*/", l):
        if group:
            locs = re.findall(r'"([^"]+)", line (\d+)', "".join(group))
            f, ln = re.findall(r'"([^"]+)", line (\d+)', group[-1])[-1]; cur = (f.split("/")[-1], int(ln))
            inner = int(re.findall(r'line (\d+)', group[0])[0]); group = []
        if cur and cur[0] == "step_kernel.cuh" and lo <= cur[1] <= hi:
            n += 1
            m = re.search(r"\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", l)
            if m: ops[m.group(2).split(".")[0]] += 1
            if "--count" not in sys.argv: print(inner, l.strip()[:110])
print("instructions:", n)
print(" ".join(f"{k}:{v}" for k, v in ops.most_common(25)))
