"""Dev tool: STL/LDL instructions of one kernel attributed to outermost step_kernel.cuh lines.
Usage: spills.py <obj.o> <kernel-regex-fragment e.g. IfLi16E>"""
import re, subprocess, sys, tempfile, os, collections
obj, frag = sys.argv[1], sys.argv[2]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cub)], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*\.text\.", txt)
blk = next(b for b in blocks if b.startswith("_ZN4hpcg18worker_step_kernel" + frag))
group, cur, cnt = [], None, collections.Counter()
for l in blk.split("\n"):
    if "//## File" in l:
        group.append(l); continue
    if re.search(r"/\*[0-9a-f]{4,}\*/", l):
        if group:
            f, ln = re.findall(r'"([^"]+)", line (\d+)', group[-1])[-1]; cur = (f.split("/")[-1], int(ln)); group = []
        m = re.search(r"\b(STL|LDL)\b", l)
        if m: cnt[(cur, m.group(1))] += 1
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "../paper_2311_04517_b200/csrc/step_kernel.cuh")).read().split("\n")
for (k, op), v in sorted(cnt.items(), key=lambda x: x[0][0][1]):
    print(f"{k[1]:5d} {op} {v:3d} | {src[k[1]-1].strip()[:90] if k[0]=='step_kernel.cuh' else k[0]}")
