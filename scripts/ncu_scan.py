"""Target for `ncu --set full`: the HBM scans of a configs[1] instance
(1M x 1000 int32): the arrival scan (row_argmin_kernel) and the full
build_index scan (seg_argmin_kernel), one launch each after a warm-up."""
import sys
sys.path.insert(0, '.')
from paper_2304_06543_b200 import solver as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
dev = S.DeviceInstance.generate(n, k, theta=0.8, pen_lo=1, pen_hi=200, mixed_families=True,
                                capacity_skew=0.5, seed=20250, device=0)
S.arrival_queue(dev)
ms, nbytes = S.bench_index_scan(dev, 2)
print(f"seg_argmin {ms:.3f} ms  {nbytes / ms / 1e6:.1f} GB/s", flush=True)
