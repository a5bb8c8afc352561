"""Solve samples of the other BASELINE shapes on one B200 (bounded |D| so each
run takes seconds to minutes): per shape the solve time, engine path (int16
tile or keys from M), counters, and the post-solve checks the library does
itself (objective recount; for small k also no negative cycle in Gamma).
usage: python scripts/gpu_shapes_solve.py [case index ...]"""
import sys, time, json
sys.path.insert(0, '.')
from paper_2304_06543_b200 import solver as S

cases = [
    # (label, n, k, theta, skew)
    ("configs[2] shape, |D| sample 100K of 4M, k=2000, capacity = demand", 100_000, 2000, 1.0, 0.0),
    ("configs[3] shape, |D| sample 200K of 2M, k=1000, skewed capacities", 200_000, 1000, 0.8, 1.0),
    ("configs[4] shape, |D| sample 20K of 10M, k=5000", 20_000, 5000, 0.8, 0.5),
]
only = sys.argv[1:]  # optional case indices
for i, (label, n, k, theta, skew) in enumerate(cases):
    if only and str(i) not in only:
        continue
    dev = S.DeviceInstance.generate(n, k, theta=theta, mixed_families=True, capacity_skew=skew, seed=3)
    t = time.time()
    try:
        rep = S.asral_solve(dev, want_assignment=False)
    except Exception as e:  # report and continue
        print(json.dumps({"case": label, "error": repr(e)}), flush=True)
        dev.close()
        continue
    el = time.time() - t
    g = S.greedy_solve(dev)
    out = {"case": label, "n": n, "k": k, "solve_s": round(el, 3),
           "device_s": round(rep.timings.device_ns / 1e9, 3), "objective": rep.objective,
           "greedy_objective": None if g is None else g.objective,
           "cycle_refines": rep.stats.cycle_refine_calls, "path_refines": rep.stats.path_refine_calls,
           "relax_rounds": rep.timings.relax_rounds, "barriers": rep.timings.grid_barriers,
           "us_per_arrival": round(rep.timings.engine_ns / 1e3 / n, 2)}
    print(json.dumps(out), flush=True)
    dev.close()
