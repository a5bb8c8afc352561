import sys
sys.path.insert(0, '.')
from paper_2304_06543_b200 import solver as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
dev = S.DeviceInstance.generate(n, 1000, theta=0.8, mixed_families=True, capacity_skew=0.5, seed=7)
rep = S.asral_solve(dev, want_assignment=False)
print("objective", rep.objective, rep.timings, S.engine_counters())
