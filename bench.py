"""Benchmark: ASRAL solve time on the BASELINE configs[1] workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one complete asral_solve (arrival scan + sort + the device
engine over every arrival + objective recount) of a synthetic
|D| = 1,000,000 x |S| = 1000 int32 instance with heterogeneous capacities
and mixed penalty families (BASELINE.json configs[1]), inputs resident in
HBM. `e2e` repeats the step through the C ABI with host buffers: upload the
pinned host cost matrix, solve, copy the assignment back.

Multi-GPU (torchrun, one process per GPU): the solve itself is a sequential
algorithm and runs as independent replicas (each rank its own instance);
the part that shards — the full cost-matrix scan behind build_index — runs
sharded by demand rows with an NCCL MIN all-reduce and is reported in the
`scan` object. Timing: CUDA events on the launching stream, barrier + sync
on both sides, max over ranks.

`--impl reference` times the reference's own CPU solver (oracle/_ref,
compiled from the reference sources; the C port when absent) on this box's
host cores on a bounded sample of the same workload (the first arrivals of
the same instance), extrapolated linearly to the full arrival count.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "ASRAL solve time (s) and cost-matrix scan GB/s vs HBM peak at 1/2/4/8 B200"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=1)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=1_000_000)
    p.add_argument("--k", type=int, default=1000)
    p.add_argument("--seed", type=int, default=20250)
    p.add_argument("--ref-seconds", type=float, default=20.0,
                   help="CPU budget of the bounded reference sample")
    return p.parse_args()


def engine_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of one cluster_engine_kernel
    launch (4096 arrivals) from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "engine_traffic.json")) as f:
            t = json.load(f)
        return int(t["dram_bytes_per_launch"]), t.get("source", "")
    except Exception:
        return None, ""


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons}


def dist_setup(n_gpus):
    import torch
    import torch.distributed as dist
    if n_gpus > 1 or "RANK" in os.environ:
        dist.init_process_group("nccl")
        rank = dist.get_rank()
        world = dist.get_world_size()
        local = int(os.environ.get("LOCAL_RANK", rank))
    else:
        rank, world, local = 0, 1, 0
    torch.cuda.set_device(local)
    return rank, world, local


def barrier():
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
        torch.cuda.synchronize()


def max_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2304_06543_b200 import solver as S
    from paper_2304_06543_b200.instance import DescHolder
    from paper_2304_06543_b200.sharded import combine_min_transfer, shard_rows
    from paper_2304_06543_b200 import _abi
    import ctypes as C

    rank, world, local = dist_setup(a.gpus)
    n, k = a.n, a.k
    # each rank: its own replica instance of configs[1] (weak scaling)
    dev = S.DeviceInstance.generate(n, k, theta=0.8, pen_lo=1, pen_hi=200, mixed_families=True,
                                    capacity_skew=0.5, seed=a.seed + rank, device=local)
    stream = torch.cuda.current_stream()

    # ---- device-resident solve: warmup + timed steps ----
    for _ in range(a.warmup):
        S.asral_solve(dev, want_assignment=False)
    barrier()
    launches0 = S.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reports = []
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        t0 = time.perf_counter()
        for _ in range(a.steps):
            reports.append(S.asral_solve(dev, want_assignment=False))
        ev1.record(stream)
        barrier()
        wall = time.perf_counter() - t0
    launches = S.launch_count() - launches0
    # device time: CUDA events recorded by the library on the stream it
    # launches on, around each whole solve (report.timings.device_ns)
    dev_s = sum(r.timings.device_ns for r in reports) / 1e9
    step_s = max_over_ranks(dev_s / a.steps)
    rep = reports[-1]
    objective = rep.objective

    # ---- e2e through the C ABI with host buffers ----
    host = dev.costs()                                   # the instance, on the host
    pinned = torch.from_numpy(host).pin_memory()
    cap, fam, off, par = dev.centers()
    desc = _abi.InstanceDesc(n, k, C.cast(pinned.data_ptr(), _abi.I32P),
                             cap.ctypes.data_as(_abi.I64P), fam.ctypes.data_as(_abi.I32P),
                             off.ctypes.data_as(_abi.I64P), par.ctypes.data_as(_abi.I64P))
    assign_host = torch.empty(n, dtype=torch.int32).pin_memory()
    e2e_times = []
    barrier()
    for _ in range(max(1, min(a.steps, 2))):
        t0 = time.perf_counter()
        h = C.c_void_p()
        S._check(S._lib.lbdd_b200_instance_create(C.byref(desc), local, C.byref(h)))
        oc, keep = S.SolverOptions().to_c()
        r = _abi.SolveReportC()
        S._check(S._lib.lbdd_b200_solve(h, 0, C.byref(oc), C.byref(r),
                                        C.cast(assign_host.data_ptr(), _abi.I32P), None))
        S._check(S._lib.lbdd_b200_instance_destroy(h))
        e2e_times.append(time.perf_counter() - t0)
        assert r.objective == objective, "e2e objective differs from the resident solve"
    e2e_s = max_over_ranks(statistics.mean(e2e_times))

    # ---- the sharded full-matrix scan (build_index) ----
    bc, _, _ = S.arrival_queue(dev)
    ms, nbytes = S.bench_index_scan(dev, 5)
    scan_gbs = nbytes / (ms / 1e3) / 1e9
    # sharded: each rank scans 1/world of its rows, MIN all-reduce over NCCL
    row0, rows = shard_rows(n, world, rank)
    d_assign = torch.from_numpy(bc).cuda()
    part = torch.empty(k * k, dtype=torch.int64, device="cuda")
    for _ in range(3):
        S.build_index_device(dev, d_assign.data_ptr(), part.data_ptr(), row0, rows,
                             stream.cuda_stream)
        combine_min_transfer(part)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        S.build_index_device(dev, d_assign.data_ptr(), part.data_ptr(), row0, rows,
                             stream.cuda_stream)
        combine_min_transfer(part)
    e1.record(stream)
    barrier()
    shard_ms = max_over_ranks(e0.elapsed_time(e1) / 5)

    peak, peak_kind = peaks()
    # dominant kernel: cluster_engine_kernel (the arrival loop). Algorithmic
    # bytes: the cost row of every arrival (4k B) and of every
    # applied transfer (4k B, its keys into the k-1 lists of the new row).
    # Duration: CUDA events around each engine launch on the library's stream.
    eng_launches = max(1, rep.timings.engine_launches)
    eng_ns_per_launch = rep.timings.engine_ns / eng_launches
    eng_bytes_per_launch = (n + rep.stats.transfers_applied) * k * 4 / eng_launches
    engine_gbs = eng_bytes_per_launch / max(eng_ns_per_launch, 1)
    row_gbs = n * k * 4 / max(rep.timings.row_scan_ns, 1)
    rounds = rep.timings.relax_rounds
    line = {
        "metric": "asral_solve_time_s",
        "baseline_metric": BASELINE_METRIC,
        "value": round(step_s, 4),
        "unit": "s",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": round(step_s * 1e3, 2),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic (device-generated euclidean costs, seeded)",
        "config": {"workload": "configs[1]: |D|=1M x |S|=1000 int32, theta 0.8, skewed capacities, "
                               "mixed penalty families" if (n, k) == (1_000_000, 1000)
                   else f"|D|={n} x |S|={k} int32 (NOT the configs[1] size)",
                   "n_demands": n, "n_centers": k, "parallelism": f"replicas x{world} (solve), "
                   f"rows sharded x{world} (scan)", "l2": "inputs (4 GB) larger than L2",
                   "objective": objective},
        "e2e": {"value": round(e2e_s, 4), "unit": "s", "h2d_bytes_per_step": int(n * k * 4),
                "d2h_bytes_per_step": int(n * 4)},
        "gpu_launches": int(launches // a.steps),
        "roofline": {"kernel": "cluster_engine_kernel", "bound": "hbm",
                     "achieved": round(engine_gbs, 3), "peak": peak, "unit": "GB/s",
                     "frac": round(engine_gbs / peak, 6), "traffic": engine_traffic()[0],
                     "traffic_source": engine_traffic()[1],
                     "launches_per_step": eng_launches,
                     "ms_per_launch": round(eng_ns_per_launch / 1e6, 3),
                     "share_of_step": round(rep.timings.engine_ns / max(rep.timings.device_ns, 1), 4),
                     "note": f"peak {peak_kind} (MEASURED_PEAKS.json hbm_gbs); latency-bound: "
                             f"{rep.timings.grid_barriers} cluster barriers, {rounds} relaxation "
                             "rounds per solve; bytes = 4k per arrival + 4k per applied transfer"},
        "scan": {"kernel": "seg_argmin_kernel (build_index full-matrix scan)",
                 "ms": round(ms, 4), "achieved": round(scan_gbs, 1), "peak": peak, "unit": "GB/s",
                 "frac": round(scan_gbs / peak, 4), "bytes": nbytes,
                 "sharded_ms_incl_allreduce": round(shard_ms, 4), "sharded_ranks": world},
        "arrival_scan": {"kernel": "row_argmin_kernel", "ms": round(rep.timings.row_scan_ns / 1e6, 4),
                         "achieved": round(row_gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(row_gbs / peak, 4), "bytes": n * k * 4},
        "host_wall_s_per_step": round(wall / a.steps, 4),
        "stats": {"cycle_refines": rep.stats.cycle_refine_calls,
                  "path_refines": rep.stats.path_refine_calls,
                  "cycles_removed": rep.stats.negative_cycles_removed,
                  "paths_removed": rep.stats.negative_paths_removed,
                  "relax_rounds": rounds, "grid_barriers": rep.timings.grid_barriers},
        "clocks": clocks.summary(),
    }
    if rank == 0:
        line["cpu_baseline"] = cpu_baseline(dev, a, host, cap, fam, off, par)
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def _problem(host, cap, fam, off, par):
    from paper_2304_06543_b200.instance import ProblemInstance
    params = [list(par[off[i]:off[i + 1]]) for i in range(len(cap))]
    return ProblemInstance.from_arrays(host, cap, fam, params)


def cpu_sample(problem, budget_s):
    """Bounded sample of the reference's asral main loop on this host: the
    first arrivals of the instance, grown until the loop alone takes about
    budget_s / 2. Sequential: the reference's para-ASRAL WorkerPool
    (parallel.hpp:31-124) can lose its done_cv_ wake-up and hang (DESIGN.md
    §6), so the stock single-threaded asral_solve loop is what is timed."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    lib, kind = pyoracle.reference(), "reference"
    if lib is None:
        lib, kind = pyoracle.oracle(), "port"
    arrivals = 16
    while True:
        ns, done, setup = lib.asral_sample(problem, arrivals, 1)
        loop_s = (ns - setup) / 1e9
        if loop_s >= budget_s / 2 or done >= problem.n:
            break
        arrivals = int(arrivals * min(8.0, max(1.5, budget_s / 2 / max(loop_s, 1e-3))))
    # estimate of the whole solve: setup (arrival queue, empty index) + the
    # loop's per-arrival rate over every arrival. A lower bound: later
    # arrivals meet fuller transfer heaps and overloaded centers.
    est = setup / 1e9 + loop_s / done * problem.n
    return kind, 1, est, done, ns / 1e9, setup / 1e9


def cpu_baseline(dev, a, host, cap, fam, off, par):
    try:
        problem = _problem(host, cap, fam, off, par)
        kind, workers, est, done, secs, setup = cpu_sample(problem, a.ref_seconds)
        return {"value": round(est, 1), "unit": "s", "cores": workers, "kind": kind,
                "sample": f"first {done} of {a.n} arrivals of the same instance ({secs:.1f} s "
                          f"incl. {setup:.1f} s setup), extrapolated linearly (lower bound)"}
    except Exception as e:  # keep the GPU line even if the host sample fails
        return {"value": None, "unit": "s", "cores": 1, "kind": "reference",
                "sample": f"failed: {e}"}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2304_06543_b200 import solver as S
    dev = S.DeviceInstance.generate(a.n, a.k, theta=0.8, pen_lo=1, pen_hi=200, mixed_families=True,
                                    capacity_skew=0.5, seed=a.seed, device=0)
    host = dev.costs()
    cap, fam, off, par = dev.centers()
    dev.close()
    problem = _problem(host, cap, fam, off, par)
    vals = []
    for step in range(a.warmup + a.steps):
        budget = a.ref_seconds / max(1, a.steps) if step >= a.warmup else 1.0
        kind, w, est, done, secs, setup = cpu_sample(problem, budget)
        if step >= a.warmup:
            vals.append(est)
    v = round(statistics.mean(vals), 1)
    line = {"impl": "reference", "metric": "asral_solve_time_s", "value": v, "unit": "s",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "higher_is_better": False,
            "scaling": "weak", "dtype": "int64", "data": "synthetic (same instance as ours)",
            "config": {"workload": "configs[1]: |D|=1M x |S|=1000", "n_demands": a.n,
                       "n_centers": a.k},
            "cpu_baseline": {"value": v, "unit": "s", "cores": w, "kind": kind,
                             "sample": f"first {done} of {a.n} arrivals per step ({secs:.1f} s "
                                       f"incl. {setup:.1f} s setup), sequential asral loop "
                                       "(para-ASRAL's pool can deadlock), extrapolated linearly "
                                       "(lower bound)"},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
