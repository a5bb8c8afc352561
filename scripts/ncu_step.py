"""ncu target: ONE bench step (one asral_solve of configs[1], 1M x 1000
int32, the bench's instance recipe) followed by the build_index scan that
bench.py reports. usage: python scripts/ncu_step.py [n] [k]"""
import sys
sys.path.insert(0, '.')
from paper_2304_06543_b200 import solver as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
dev = S.DeviceInstance.generate(n, k, theta=0.8, pen_lo=1, pen_hi=200, mixed_families=True,
                                capacity_skew=0.5, seed=20250, device=0)
rep = S.asral_solve(dev, want_assignment=False)
t = rep.timings
print(f"solve {n}x{k}: objective {rep.objective} device {t.device_ns / 1e9:.3f}s "
      f"engine {t.engine_ns / 1e9:.3f}s in {t.engine_launches} launches, "
      f"row scan {t.row_scan_ns / 1e6:.3f} ms", flush=True)
ms, nbytes = S.bench_index_scan(dev, 2)
print(f"seg_argmin {ms:.3f} ms  {nbytes / ms / 1e6:.1f} GB/s", flush=True)
