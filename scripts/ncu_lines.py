"""Warp-stall samples per CUDA source line of an ncu report (read here, after
gpurun brings the .ncu-rep back): python scripts/ncu_lines.py REP [TOP]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, src, fname = {}, {}, "?"
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if not r[0].strip():
        continue  # a SASS row under its source line (already counted there)
    try:
        v = int(r[iS])
    except ValueError:
        continue
    key = (fname, int(r[0]))
    agg[key] = agg.get(key, 0) + v
    src[key] = r[1].strip()[:100]
tot = sum(agg.values()) or 1
print("total samples", tot)
for key, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:8d} {100 * v / tot:5.1f}%  {key[0]}:{key[1]:<5d} {src[key]}")
