"""Summarise an ncu launch list (gpu__time_duration.sum per launch, --csv)
into per-kernel launch counts, total time and share.
usage: python scripts/launch_summary.py launches.csv"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
mult = {'ns': 1e-9, 'nsecond': 1e-9, 'us': 1e-6, 'usecond': 1e-6, 'ms': 1e-3, 'msecond': 1e-3,
        's': 1, 'second': 1}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi or not r[vi]:
        continue
    name = r[ki].split('(')[0].replace('void ', '')[:70]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(',', '')) * mult[r[ui]]
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':70s} {'launches':>8s} {'total s':>10s} {'share':>8s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:70s} {v[0]:8d} {v[1]:10.4f} {100 * v[1] / tot:7.3f}%")
print(f"{'total':70s} {sum(v[0] for v in agg.values()):8d} {tot:10.4f}")
