import os, sys, time
sys.path.insert(0, '.')
from paper_2304_06543_b200 import solver as S
n, k = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (20000, 1000)
dev = S.DeviceInstance.generate(n, k, theta=0.8, mixed_families=True, capacity_skew=0.5, seed=7)
t = time.time(); rep = S.asral_solve(dev, want_assignment=False); el = time.time() - t
c = S.engine_counters()
cyc = c.pop("cycles")
print(n, k, rep.objective, "%.2fs" % el, "dev %.2fs" % (rep.timings.device_ns / 1e9), "barriers", rep.timings.grid_barriers)
print("  ", c)
tot = sum(cyc.values())
for kk, v in cyc.items():
    print("   %-12s %5.1f%%  %8.1f ms" % (kk, 100 * v / max(tot, 1), v / 1.9e6))
