import sys, time
sys.path.insert(0, '.')
from paper_2304_06543_b200 import solver as S
for n, k in [(20000, 1000), (10000, 100)]:
    dev = S.DeviceInstance.generate(n, k, theta=0.8, mixed_families=True, capacity_skew=0.5, seed=7)
    t = time.time(); rep = S.asral_solve(dev, want_assignment=False); el = time.time() - t
    print(n, k, rep.objective, "%.2fs" % el, rep.stats, flush=True)
    print("  ", S.engine_counters(), "rounds", rep.timings.relax_rounds, "barriers", rep.timings.grid_barriers, flush=True)
