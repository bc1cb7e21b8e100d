"""Dev tool: executed warp-instructions by SASS opcode (optionally restricted to a source-line range
of one file) from an ncu --set full report with --import-source. usage:
python tools/ncu_opcodes.py rep.ncu-rep [file.cuh a-b]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
flt = (sys.argv[2], *map(int, sys.argv[3].split("-"))) if len(sys.argv) > 3 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, line, agg = None, None, None, {}
for row in csv.reader(io.StringIO(txt)):
    if not row:
        continue
    if row[0] in ("File Path", "File Name"):
        cur = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None:
        continue
    if row[0].isdigit():
        line = int(row[0])
        continue
    if row[0] == "" and len(row) > 4 and row[2].startswith("0x"):
        if flt and not (cur == flt[0] and flt[1] <= (line or 0) <= flt[2]):
            continue
        d = dict(zip(hdr[2:], row[2:]))
        try:
            n = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            n = 0
        sass = row[3].strip().split()
        op = sass[1] if sass and sass[0].startswith("@") and len(sass) > 1 else (sass[0] if sass else "?")
        op = op.split(".")[0]
        agg[op] = agg.get(op, 0) + n
tot = sum(agg.values())
print(f"total {tot}")
for op, n in sorted(agg.items(), key=lambda x: -x[1])[:30]:
    print(f"  {op:10s} {n:>11d} {100 * n / max(tot, 1):5.1f}%")
