"""Dev tool: per-source-line instructions executed and warp-stall samples of an ncu --set full report
(needs -lineinfo and --import-source), summed over line ranges. usage:
python tools/ncu_phases.py rep.ncu-rep file.cuh name:a-b [name:a-b ...]  (prints top lines if no ranges)"""
import csv
import io
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
ranges = [(a.split(":")[0], *map(int, a.split(":")[1].split("-"))) for a in sys.argv[3:]]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, rows = None, None, []
for row in csv.reader(io.StringIO(txt)):
    if not row:
        continue
    if row[0] in ("File Path", "File Name"):
        cur = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0].isdigit():
        continue
    d = dict(zip(hdr[2:], row[2:]))
    def num(k):
        try:
            return int(d.get(k, "0") or 0)
        except ValueError:
            return 0
    rows.append((cur, int(row[0]), num("Instructions Executed"), num("Warp Stall Sampling (All Samples)"),
                 row[1][:90], {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not" not in k and v.isdigit() and int(v) > 0}))
tot_i = sum(r[2] for r in rows)
tot_s = sum(r[3] for r in rows)
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
if ranges:
    for nm, a, b in ranges:
        sel = [r for r in rows if r[0] == fname and a <= r[1] <= b]
        i = sum(r[2] for r in sel); s = sum(r[3] for r in sel)
        st = {}
        for r in sel:
            for k, v in r[5].items():
                st[k] = st.get(k, 0) + v
        top = sorted(st.items(), key=lambda x: -x[1])[:4]
        print(f"{nm:12s} lines {a}-{b}: instr {i:>11d} ({100*i/tot_i:5.1f}%)  samples {s:>7d} ({100*s/tot_s:5.1f}%)  "
              + " ".join(f"{k[6:]}={v}" for k, v in top))
    other = [r for r in rows if r[0] != fname]
    print(f"{'other files':12s} instr {sum(r[2] for r in other)} samples {sum(r[3] for r in other)}")
else:
    for r in sorted(rows, key=lambda r: -r[3])[:40]:
        print(f"{r[0]}:{r[1]:5d} instr {r[2]:>9d} samples {r[3]:>6d} {r[4]}")
if "--files" in sys.argv or True:
    agg = {}
    for r in rows:
        a = agg.setdefault(r[0], [0, 0])
        a[0] += r[2]; a[1] += r[3]
    for f, (i, s) in sorted(agg.items(), key=lambda x: -x[1][1])[:8]:
        print(f"  file {f:40s} instr {i:>11d} samples {s:>7d}")
    oth = sorted([r for r in rows if r[0] != fname], key=lambda r: -r[3])[:12]
    for r in oth:
        print(f"  {r[0]}:{r[1]} instr {r[2]} samples {r[3]} {r[4][:60]} {sorted(r[5].items(), key=lambda x:-x[1])[:3]}")
st = {}
for r in rows:
    if r[0] in ("helpers.h", "sm_90_rt.hpp") :
        continue
    for k, v in r[5].items():
        st[k] = st.get(k, 0) + v
print("stalls (all lines):", " ".join(f"{k[6:]}={v}" for k, v in sorted(st.items(), key=lambda x: -x[1])))
