import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np
import pyoracle as po
from paper_2304_06543_b200 import solver as S, SolverOptions
O = po.oracle()
rng = po.Mt19937_64(61)
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 60):
    n = 1 + rng() % 40; k = 1 + rng() % 6
    inst = po.random_instance(rng, n=n, k=k, total_capacity=(rng() % (n+1)) if it % 2 else -1)
    asg = np.array([rng() % k for _ in range(n)], np.int32)
    print("it", it, n, k, flush=True) if "-v" in sys.argv else None
    for solver in ["asral", "strict"]:
        for fix in [False, True]:
            opts = SolverOptions(refine_to_fixpoint=fix, check_invariants=(it % 3 == 0))
            b = O.solve(inst, solver, opts)
            try:
                a = S.solve(inst, solver, opts)
                ok = a.objective == b.objective and (a.assignment == b.assignment).all()
            except Exception as e:
                ok = False; a = e
            if not ok:
                print("FAIL it", it, solver, fix, "n", n, "k", k, a if isinstance(a, Exception) else a.objective, b.objective, flush=True)
                sys.exit(1)
print("all ok")
