"""Quick GPU sanity run: device path vs the oracle on small cases."""
import sys, time, traceback
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np
import pyoracle as po
from paper_2304_06543_b200 import solver as S, SolverOptions
O = po.oracle()
print(S.version(), "devices", S.device_count(), flush=True)

def cmp(tag, a, b):
    ok = (a.objective == b.objective and (a.assignment == b.assignment).all() and a.stats == b.stats
          and a.strict_surcharge == b.strict_surcharge)
    if not ok:
        print("MISMATCH", tag, a.objective, b.objective, a.stats, b.stats, flush=True)
    return ok

# worked cycle example
inst = po.ProblemInstance([po.ServiceCenter(s, 2, po.PenaltySpec.constant(5)) for s in range(4)],
    np.array([[10,6,20,20],[20,10,7,20],[20,20,10,7],[7,20,20,10]], np.int32))
print("cycle:", S.negative_cycle_refine(inst, [0,1,2,3], 0)[:3], O.refine(inst, 0, 0, [0,1,2,3])[:3], flush=True)
# lowest cost path random
rng = po.Mt19937_64(43); bad = 0; tot = 0
for it in range(200):
    k = 2 + rng() % 5
    nodes = k + 1
    w = np.full((k, nodes), po.NO_EDGE, np.int64)
    anchor = rng() % k
    for u in range(k):
        for v in range(k):
            if u == v: continue
            if rng() % 10 < 6:
                w[u, k if v == anchor else v] = (rng() % 41) - 20
    try:
        a = O.lowest_cost_path(w, anchor)
    except Exception as e:
        a = type(e).__name__
    try:
        b = S.lowest_cost_path(w, anchor)
    except Exception as e:
        b = type(e).__name__
    tot += 1
    same = (a == b) if isinstance(a, str) or a is None or isinstance(b, str) or b is None else (
        a[0] == b[0] and (a[1] == b[1]).all() and (a[2] == b[2]).all() and (a[3] == b[3]).all())
    if not same:
        bad += 1
        if bad < 3: print("LCP mismatch", a, b)
print("lcp bad", bad, "of", tot, flush=True)
rng = po.Mt19937_64(61); bad = 0
t0 = time.time()
for it in range(60):
    n = 1 + rng() % 40; k = 1 + rng() % 6
    inst = po.random_instance(rng, n=n, k=k, total_capacity=(rng() % (n+1)) if it % 2 else -1)
    asg = np.array([rng() % k for _ in range(n)], np.int32)
    if not (S.build_index(inst, asg) == O.build_index(inst, asg)).all():
        bad += 1; print("build_index mismatch", it)
    for solver in ["asral", "strict", "greedy"]:
        for fix in [False, True]:
            opts = SolverOptions(refine_to_fixpoint=fix, check_invariants=(it % 3 == 0))
            try:
                a = S.solve(inst, solver, opts)
            except Exception:
                traceback.print_exc(); bad += 1; continue
            b = O.solve(inst, solver, opts)
            if not cmp((it, solver, fix), a, b): bad += 1
print("solve bad", bad, "time %.1f" % (time.time() - t0), flush=True)
inst = O.generate(42, 10000, 100.0, 0.8, 1, 200)
t = time.time(); a = S.asral_solve(inst); ta = time.time() - t
b = O.solve(inst, "asral")
print("config0", cmp("cfg0", a, b), a.objective, b.objective, "gpu %.2fs" % ta, a.timings, flush=True)
dev = S.DeviceInstance.generate(1000000, 1000, theta=0.8, mixed_families=True, capacity_skew=0.5, seed=7)
ms, nb = S.bench_index_scan(dev, 5)
print("index scan 1M x 1000: %.3f ms  %.1f GB/s" % (ms, nb / ms / 1e6), flush=True)
t = time.time(); g = S.greedy_solve(dev); print("greedy", g.objective, "%.2fs" % (time.time()-t), flush=True)
t = time.time()
rep = S.asral_solve(dev, want_assignment=False)
print("asral 1M x 1000:", rep.objective, "%.2fs" % (time.time() - t), rep.stats, rep.timings, flush=True)
