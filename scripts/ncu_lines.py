"""Aggregate an ncu source page (cuda,sass CSV) into per-source-line warp
stall samples: top lines and their dominant stall reasons.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
       python scripts/ncu_lines.py s.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
col = {h: i for i, h in enumerate(hdr)}
samp = col["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
file_lines = {}
cur = None
agg = collections.defaultdict(lambda: collections.Counter())
tot = 0
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr):
        if r and r[0] == "File Path":
            pass
        continue
    if r[0]:
        cur = int(r[0]) if r[0].isdigit() else None
        file_lines[cur] = r[1]
        continue
    if cur is None:
        continue
    try:
        n = float(r[samp] or 0)
    except ValueError:
        continue
    tot += n
    agg[cur]["_"] += n
    for h in stalls:
        v = r[col[h]]
        if v and v != "0":
            agg[cur][h] += float(v)
print(f"total samples {tot:.0f}")
for ln, c in sorted(agg.items(), key=lambda x: -x[1]["_"])[:top]:
    st = sorted(((v, k) for k, v in c.items() if k != "_"), reverse=True)[:3]
    sts = ", ".join(f"{k[6:]} {100 * v / c['_']:.0f}%" for v, k in st)
    print(f"{100 * c['_'] / tot:5.1f}% L{ln:<5d} {file_lines.get(ln, '')[:70]:70s} | {sts}")
