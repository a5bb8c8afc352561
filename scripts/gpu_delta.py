import os, sys, time, subprocess
for d in sys.argv[1:]:
    env = dict(os.environ, LBDD_B200_DELTA=d)
    out = subprocess.run([sys.executable, "-c", """
import sys, time
sys.path.insert(0, '.')
from paper_2304_06543_b200 import solver as S
dev = S.DeviceInstance.generate(20000, 1000, theta=0.8, mixed_families=True, capacity_skew=0.5, seed=7)
t = time.time(); rep = S.asral_solve(dev, want_assignment=False); el = time.time() - t
c = S.engine_counters()
print(rep.objective, '%.2fs' % el, 'rounds', rep.timings.relax_rounds, {kk: v for kk, v in c.items() if kk != 'cycles'})
"""], env=env, capture_output=True, text=True)
    print("delta", d, out.stdout.strip(), out.stderr.strip()[-300:], flush=True)
