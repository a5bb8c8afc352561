"""Latency floor of the cluster engine's per-round primitive: one cluster
barrier + the DSMEM exchange of every CTA's published scalars (mode 0), and
the same with 128 remote frontier entries staged per round (mode 1), on a
16-CTA cluster of 512 threads (cluster_exchange_bench in cluster.cu).
Writes gpurun_out/cluster_latency.json (copied to profiles/ when judged)."""
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2304_06543_b200 import solver as S  # noqa: E402

S._lib.lbdd_b200_debug_exchange_cycles.restype = C.c_longlong
clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                     capture_output=True, text=True).stdout.strip().split("\n")[0]
mhz = float(clk) if clk.replace(".", "").isdigit() else 1965.0
out = {}
for cs in (16, 8):
    for mode in (0, 1, 2, 4, 8):
        cyc = min(S._lib.lbdd_b200_debug_exchange_cycles(cs, 20000, mode) for _ in range(3))
        out[f"cs{cs}_mode{mode}_cycles"] = cyc
mx = 1965.0
res = {"barrier_exchange_cycles": out["cs16_mode0_cycles"],
       "barrier_exchange_us": round(out["cs16_mode0_cycles"] / mx, 4),
       "barrier_exchange_staged_us": round(out["cs16_mode1_cycles"] / mx, 4),
       "relaxed_barrier_us": round(out["cs16_mode4_cycles"] / mx, 4),
       "st_async_mbarrier_us": round(out["cs16_mode8_cycles"] / mx, 4),
       "all": out, "sm_mhz_sampled": mhz,
       "source": "scripts/latency_floor.py: cluster_exchange_bench (cluster.cu), 16 CTAs x 512 "
                 "threads, clock64 cycles per round / 1965 MHz"}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "cluster_latency.json"), "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res))
