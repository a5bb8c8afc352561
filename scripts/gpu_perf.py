import sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np
import pyoracle as po
from paper_2304_06543_b200 import solver as S, SolverOptions
O = po.oracle()
inst = O.generate(42, 10000, 100.0, 0.8, 1, 200)
t = time.time(); a = S.asral_solve(inst); ta = time.time() - t
b = O.solve(inst, "asral")
print("config0 ok", a.objective == b.objective and (a.assignment == b.assignment).all(), "gpu %.2fs" % ta, a.timings, flush=True)
print("  us/barrier %.2f" % (a.timings.total_ns / 1e3 / a.timings.grid_barriers))
for n in [20000, 100000]:
    dev = S.DeviceInstance.generate(n, 1000, theta=0.8, mixed_families=True, capacity_skew=0.5, seed=7)
    t = time.time()
    rep = S.asral_solve(dev, want_assignment=False)
    el = time.time() - t
    print(f"asral {n} x 1000:", rep.objective, "%.2fs" % el, rep.stats, rep.timings, flush=True)
    print("  us/barrier %.2f  rounds/refine %.1f" % (el * 1e6 / rep.timings.grid_barriers,
          rep.timings.relax_rounds / (rep.stats.cycle_refine_calls + rep.stats.path_refine_calls)), flush=True)
