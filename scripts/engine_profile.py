"""Cluster-engine phase profile of one solve (LBDD_B200_PROF=1): lead-thread
cycles per phase, per-CTA work / wait cycles, search statistics; optional
sweeps of the Δ-stepping widths. Diagnostics only.

usage: python scripts/engine_profile.py [--n N] [--k K] [--delta-path 1,4,16]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth_instances as SI  # noqa: E402
from paper_2304_06543_b200 import solver as S  # noqa: E402

PHASES = {0: "T1 (apply lists)", 1: "relax", 2: "collect", 3: "round exchange",
          4: "insert + first round", 5: "cycle search tail", 6: "pi repair apply",
          7: "path bound", 8: "path search tail", 9: "round start / pre-reconstruct",
          10: "reconstruct", 11: "apply tail", 12: "apply exchanges", 13: "T3 rescans",
          14: "arrival start"}

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=200_000)
p.add_argument("--k", type=int, default=1000)
p.add_argument("--seed", type=int, default=20250)
p.add_argument("--theta", default="8/10")
p.add_argument("--delta-path", default="")
p.add_argument("--delta", default="")
p.add_argument("--noprof", action="store_true")
a = p.parse_args()
tn, td = (int(x) for x in a.theta.split("/"))
spec = SI.SynthSpec(a.n, a.k, seed=a.seed, theta_num=tn, theta_den=td)
dev = S.DeviceInstance.from_spec(spec)
if not a.noprof:
    os.environ["LBDD_B200_PROF"] = "1"
runs = [("", "")]
if a.delta_path or a.delta:
    runs = [(dm, dp) for dm in (a.delta.split(",") if a.delta else [""])
            for dp in (a.delta_path.split(",") if a.delta_path else [""])]
for dm, dp in runs:
    for var, val in (("LBDD_B200_DELTA", dm), ("LBDD_B200_DELTA_PATH", dp)):
        if val:
            os.environ[var] = val
        else:
            os.environ.pop(var, None)
    t = time.time()
    rep = S.asral_solve(dev, want_assignment=False)
    el = time.time() - t
    tm = rep.timings
    c = np.zeros(72, np.int64)
    S._lib.lbdd_b200_engine_counters(c.ctypes.data_as(S._abi.I64P))
    c = [int(x) for x in c]
    print(f"== {spec.name()} delta={dm or 'def'} delta_path={dp or 'def'}: objective {rep.objective} "
          f"wall {el:.2f}s engine {tm.engine_ns / 1e9:.3f}s rounds {tm.relax_rounds} "
          f"barriers {tm.grid_barriers} ({tm.engine_ns / max(1, tm.grid_barriers) / 1e3:.2f} us/barrier, "
          f"{tm.grid_barriers / a.n:.2f}/arrival)", flush=True)
    print("  stats", rep.stats, flush=True)
    print(f"  searches c/p/r {c[0]}/{c[1]}/{c[2]} empty {c[3]}/{c[4]}/{c[5]} frontier {c[6]}/{c[7]}/{c[8]} "
          f"pruned {c[9]} rounds {c[10]}/{c[11]}/{c[12]}", flush=True)
    if a.noprof:
        continue
    tot = sum(c[16 + i] for i in range(15)) or 1
    for i in range(15):
        v = c[16 + i]
        if v:
            print(f"  {PHASES[i]:32s} {v / 1e9:8.3f} Gcyc {100 * v / tot:5.1f}%  {v / a.n:9.0f} cyc/arrival",
                  flush=True)
    work = c[40:56]
    wait = c[56:72]
    print("  per-CTA work Gcyc", [round(x / 1e9, 2) for x in work], flush=True)
    print("  per-CTA wait Gcyc", [round(x / 1e9, 2) for x in wait], flush=True)
    print(f"  rescans calls {c[32]} full {c[33]} rowmode {c[34]} candidates {c[35]} members {c[36]} "
          f"pairs {c[37]}", flush=True)
