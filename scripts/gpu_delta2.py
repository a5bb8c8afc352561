"""Sweep Δ (cycle/repair searches) and Δ_path (penalty-path searches) on one
instance; every setting must give the same objective (exact search)."""
import os, sys, subprocess
n = int(sys.argv[1]); k = int(sys.argv[2])
for spec in sys.argv[3:]:
    d, dp, *ch = spec.split(",")
    env = dict(os.environ, LBDD_B200_DELTA=d, LBDD_B200_DELTA_PATH=dp, LBDD_B200_PROF=os.environ.get("LBDD_B200_PROF", "1"))
    if ch:
        env["LBDD_B200_CHUNK"] = ch[0]
    out = subprocess.run([sys.executable, "-c", f"""
import sys, time
sys.path.insert(0, '.')
from paper_2304_06543_b200 import solver as S
dev = S.DeviceInstance.generate({n}, {k}, theta=0.8, mixed_families=True, capacity_skew=0.5, seed=7)
t = time.time(); rep = S.asral_solve(dev, want_assignment=False); el = time.time() - t
c = S.engine_counters()
tot = sum(c['cycles'].values()) or 1
print(rep.objective, '%.2fs' % el, 'rounds', rep.timings.relax_rounds, 'barriers', rep.timings.grid_barriers,
      {{kk: v for kk, v in c.items() if kk not in ('cycles',)}},
      {{p: round(v / tot, 3) for p, v in c['cycles'].items()}})
"""], env=env, capture_output=True, text=True)
    print("delta", d, "delta_path", dp, "chunk", ch, out.stdout.strip(), out.stderr.strip()[-300:], flush=True)
