"""HBM scans at the BASELINE shapes that fit one B200: the arrival scan
(row_argmin_kernel, from the solve's report) and the build_index scan
(seg_argmin_kernel), in GB/s of algorithmic bytes vs the measured HBM peak.
configs[4] (10M x 5000, 200 GB) is sharded 8 ways by demand rows; one rank's
shard is 1.25M x 5000 (25 GB) and is what a single GPU scans.
usage: python scripts/scan_shapes.py [json]"""
import json, os, sys
sys.path.insert(0, '.')
from paper_2304_06543_b200 import solver as S
peak = json.load(open('MEASURED_PEAKS.json'))['hbm_gbs'] if os.path.exists('MEASURED_PEAKS.json') else 6650.0
shapes = [("configs[1]", 1_000_000, 1000), ("configs[2]", 4_000_000, 2000),
          ("configs[3] shape", 2_000_000, 1000), ("configs[4] per-rank shard (1/8)", 1_250_000, 5000)]
out = []
for name, n, k in shapes:
    dev = S.DeviceInstance.generate(n, k, theta=0.8, pen_lo=1, pen_hi=200, mixed_families=True,
                                    capacity_skew=0.5, seed=7, device=0)
    g = S._solve(dev, S._abi.SOLVER_GREEDY, None, 0, want_assignment=False)     # arrival scan + sort + recount
    S._solve(dev, S._abi.SOLVER_GREEDY, None, 0, want_assignment=False)
    g = S._solve(dev, S._abi.SOLVER_GREEDY, None, 0, want_assignment=False)
    row_ms = g.timings.row_scan_ns / 1e6
    ms, nbytes = S.bench_index_scan(dev, 5)
    r = {"shape": name, "n": n, "k": k, "matrix_GB": round(n * k * 4 / 1e9, 2),
         "row_argmin_ms": round(row_ms, 3), "row_argmin_GBs": round(n * k * 4 / row_ms / 1e6, 1),
         "seg_argmin_ms": round(ms, 3), "seg_argmin_GBs": round(nbytes / ms / 1e6, 1), "peak": peak}
    r["row_frac"] = round(r["row_argmin_GBs"] / peak, 3)
    r["seg_frac"] = round(r["seg_argmin_GBs"] / peak, 3)
    out.append(r)
    print(json.dumps(r), flush=True)
    dev.close()
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
