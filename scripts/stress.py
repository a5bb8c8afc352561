"""Mid-size stress: device-generated instances (bench recipe, varied seeds and
shapes) solved twice on the GPU and once by the oracle (the compiled
reference when present); any mismatch or nondeterminism is printed.
usage: python scripts/stress.py SECONDS [strict]"""
import os, sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np
import pyoracle as po
from paper_2304_06543_b200 import solver as S, SolverOptions
from paper_2304_06543_b200.instance import ProblemInstance
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
modes = ["asral", "strict"] if "strict" in sys.argv else ["asral"]
O = po.reference() or po.oracle()
shapes = [(2000, 50), (5000, 100), (3000, 200), (8000, 100), (1500, 300), (20000, 64), (1000, 500)]
t_end = time.time() + budget
it = 0; bad = 0
while time.time() < t_end:
    n, k = shapes[it % len(shapes)]
    seed = 1000 + it
    theta = [0.8, 1.0, 0.6, 1.2][it % 4]
    tn, td = {0.8: (8, 10), 1.0: (1, 1), 0.6: (6, 10), 1.2: (12, 10)}[theta]
    dev = S.DeviceInstance.generate(n, k, seed=seed, theta_num=tn, theta_den=td,
                                    cap_spread=[16, 1, 64][it % 3])
    host = dev.costs(); cap, fam, off, par = dev.centers()
    params = [list(par[off[i]:off[i + 1]]) for i in range(k)]
    inst = ProblemInstance.from_arrays(host, cap, fam, params)
    for mode in modes:
        opts = SolverOptions(refine_to_fixpoint=bool(it % 2))
        try:
            a1 = S.solve(dev, mode, opts)
            a2 = S.solve(dev, mode, opts)
        except Exception as e:
            print(f"it {it} {mode} n {n} k {k} seed {seed} GPU ERROR {e!r}", flush=True); bad += 1; continue
        b = O.solve(inst, mode, opts)
        ok = a1.objective == b.objective and (a1.assignment == b.assignment).all()
        det = a1.objective == a2.objective and (a1.assignment == a2.assignment).all()
        if not (ok and det):
            bad += 1
            print(f"it {it} {mode} n {n} k {k} seed {seed} theta {theta} MISMATCH ok={ok} det={det} "
                  f"{a1.objective} {a2.objective} ref {b.objective}", flush=True)
    dev.close()
    it += 1
print(f"stress done: {it} instances, {bad} bad", flush=True)
