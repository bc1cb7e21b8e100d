"""Dev tool: warp-stall samples of an ncu --set full report aggregated by CUDA source line
(needs -lineinfo and --import-source). usage: python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, hdr, agg, total = None, None, {}, 0
for row in csv.reader(io.StringIO(txt)):
    if not row:
        continue
    if row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < len(hdr):
        continue
    if row[0]:  # a CUDA source line (its metrics aggregate the SASS below it)
        d = dict(zip(hdr[2:], row[2:]))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and v.isdigit() and int(v) > 0}
        key = (cur_file, int(row[0]))
        agg[key] = (s, row[1][:80], stalls)
        total += s
print(f"total samples {total}")
for (f, ln), (s, src, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{s:7d} {100*s/max(total,1):5.1f}% {f}:{ln:<5d} {src:80s} " + " ".join(f"{k[6:]}={v}" for k, v in top3))
