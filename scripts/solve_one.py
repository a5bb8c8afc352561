"""One (or more) device solves of a synth_instances spec, generated in HBM;
prints time, objective, stats and engine counters per solve. Also the ncu
target of scripts/gpu_profile.sh. With --golden TAG the result is compared
with tests/golden/scale/TAG.json (the reference run to completion).

usage: python scripts/solve_one.py [--n N] [--k K] [--seed S] [--theta 8/10]
                                   [--reps R] [--golden TAG] [--scan]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth_instances as SI  # noqa: E402
from paper_2304_06543_b200 import solver as S  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=1_000_000)
p.add_argument("--k", type=int, default=1000)
p.add_argument("--seed", type=int, default=20250)
p.add_argument("--theta", default="8/10")
p.add_argument("--reps", type=int, default=1)
p.add_argument("--golden", default=None)
p.add_argument("--prefix", type=int, default=0,
               help="solve only the first N arrivals (lbdd_b200_solve_prefix): large-k samples")
p.add_argument("--scan", action="store_true", help="also time the build_index scan")
p.add_argument("--road", action="store_true",
               help="configs[3]-style road-network instance (RoadSpec, host-generated)")
a = p.parse_args()
if a.golden:
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "scale", a.golden + ".json")))
    spec = SI.SynthSpec(**g["spec"])
else:
    tn, td = (int(x) for x in a.theta.split("/"))
    spec = SI.SynthSpec(a.n, a.k, seed=a.seed, theta_num=tn, theta_den=td)
print("lib", S.LIB_PATH, "engine", os.environ.get("LBDD_B200_ENGINE", "cluster"), spec.name(),
      flush=True)
if a.road:
    spec = SI.RoadSpec(a.n, a.k, seed=a.seed)
    print("road", spec.name(), flush=True)
    t0 = time.time()
    dev = S.DeviceInstance.upload(SI.road_problem(spec))
    print(f"generated + uploaded in {time.time() - t0:.1f} s", flush=True)
else:
    dev = S.DeviceInstance.from_spec(spec)
for r in range(a.reps):
    t = time.time()
    try:
        rep = (S.asral_prefix(dev, a.prefix) if a.prefix
               else S.asral_solve(dev, want_assignment=bool(a.golden)))
    except Exception as e:
        print(f"rep {r} FAILED after {time.time() - t:.1f}s: {e!r}", flush=True)
        continue
    el = time.time() - t
    tm = rep.timings
    print(f"rep {r} {spec.n}x{spec.k}: objective {rep.objective} wall {el:.2f}s device "
          f"{tm.device_ns / 1e9:.3f}s engine {tm.engine_ns / 1e9:.3f}s/{tm.engine_launches} "
          f"rounds {tm.relax_rounds} barriers {tm.grid_barriers} "
          f"row_scan {tm.row_scan_ns / 1e6:.3f}ms", flush=True)
    print("  stats", rep.stats, flush=True)
    print("  counters", S.engine_counters(), flush=True)
    if a.golden:
        ok = (rep.objective == g["objective"]
              and SI.assignment_sha256(rep.assignment) == g["assignment_sha256"])
        print(f"  golden {a.golden}: {'MATCH' if ok else 'MISMATCH'} (ref objective "
              f"{g['objective']}, ref cpu {g['cpu_seconds']} s)", flush=True)
if a.scan:
    ms, nbytes = S.bench_index_scan(dev, 3)
    print(f"seg_argmin {ms:.3f} ms {nbytes / ms / 1e6:.1f} GB/s", flush=True)
