"""Large-instance diagnostic: solve n x k (device-generated, bench's recipe)
`reps` times, printing time, objective, stats, counters; errors printed."""
import os, sys, time
sys.path.insert(0, '.')
from paper_2304_06543_b200 import solver as S
n = int(sys.argv[1]); k = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
seed = int(sys.argv[4]) if len(sys.argv) > 4 else 20250
print("lib", S.LIB_PATH, "engine", os.environ.get("LBDD_B200_ENGINE", "cluster"), flush=True)
dev = S.DeviceInstance.generate(n, k, theta=0.8, pen_lo=1, pen_hi=200, mixed_families=True,
                                capacity_skew=0.5, seed=seed, device=0)
for r in range(reps):
    t = time.time()
    try:
        rep = S.asral_solve(dev, want_assignment=False)
        el = time.time() - t
        print(f"rep {r} n {n} k {k}: objective {rep.objective} {el:.2f}s", rep.stats, rep.timings, flush=True)
        c = S.engine_counters()
        print("  counters", c, flush=True)
    except Exception as e:
        print(f"rep {r} FAILED after {time.time() - t:.1f}s: {e!r}", flush=True)
