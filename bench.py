"""Benchmark: ASRAL solve time on the BASELINE configs[1] workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one complete asral_solve (arrival scan + sort + the device
engine over every arrival + objective recount) of configs[1]: the
synth_instances.CONFIG1 instance, |D| = 1,000,000 x |S| = 1000 int32 costs,
heterogeneous capacities (80% of demand) and mixed penalty families. The
instance is generated on the HOST by synth_instances.py (not by the product
library, not by oracle/); both arms print its sha256 and solve exactly these
bytes. `value` times the solve with the matrix resident in HBM; `e2e` repeats
it through the C ABI with host buffers (pinned 4 GB upload, solve, assignment
read back).

Wall-clock budget: a configs[1] solve takes tens of seconds, so K requested
steps may not fit the driver's limit. bench.py runs at most --warmup warm-up
solves (at least 1) and as many of the --steps timed solves as fit in
--budget seconds of wall clock (always at least 1), and reports the counts
it ran as `steps`/`warmup` beside `requested_steps`/`requested_warmup`.

Multi-GPU (torchrun, one process per GPU, run_sharded): the configs[1]
matrix is split in row blocks over the ranks (each rank generates and holds
only its block); the blocks are mapped into every device with CUDA IPC, the
per-block arrival scans are all-gathered over NCCL, and the sequential
arrival loop runs replicated on every rank, reading other ranks' rows over
NVLink (paper_2304_06543_b200/sharded.py). Total work is fixed ("strong");
what scales is the matrix per GPU, not the solve time. Timing: CUDA events
on the launching stream, barrier + sync on both sides, max over ranks.
LBDD_BENCH_BACKEND=gloo (tests only) runs the ranks over gloo.

`--impl reference` times the UNMODIFIED reference solver (oracle/_ref,
compiled from the reference sources; never the product library) on this
box's host cores. A full configs[1] solve takes the reference days
(tests/golden/scale/, profiles/ref_cpu_profile_configs1.json), so each step
is a bounded sample: arrivals continued from a state the reference itself
reached mid-solve (its checkpoint, resumed through the reference's own
SolverState::from_allotment), calibrated against the reference's full-run
time profile measured in the build container (see cpu_estimate()).
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
import zlib

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "ASRAL solve time (s) and cost-matrix scan GB/s vs HBM peak at 1/2/4/8 B200"
CPU_PROFILE = os.path.join(ROOT, "profiles", "ref_cpu_profile_configs1.json")
CKPT_DIR = os.path.join(ROOT, "tests", "golden", "ckpt")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--demands", dest="n", type=int, default=None, help="override |D| (not configs[1])")
    p.add_argument("--centers", dest="k", type=int, default=None, help="override |S| (not configs[1])")
    p.add_argument("--budget", type=float, default=1380.0,
                   help="wall-clock seconds for the whole run (driver limit 1800 s)")
    p.add_argument("--ref-arrivals", type=int, default=40,
                   help="arrivals per reference sample (steady state, from the checkpoint)")
    p.add_argument("--ref-first", type=int, default=300,
                   help="arrivals of the from-scratch reference sample (solve start)")
    return p.parse_args()


def spec_of(a):
    import synth_instances as SI
    if a.n is None and a.k is None:
        return SI.CONFIG1, True
    n = a.n or SI.CONFIG1.n
    k = a.k or SI.CONFIG1.k
    return SI.SynthSpec(n, k), False


def workload_name(spec, is_cfg1):
    if is_cfg1:
        return ("configs[1]: |D|=1M x |S|=1000 int32, heterogeneous capacities (80% of demand), "
                "mixed penalty families")
    return f"|D|={spec.n} x |S|={spec.k} int32 (NOT the configs[1] size)"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 7672.0, "fallback (B200_PROFILING.md nominal HBM3e)"


def committed_json(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return None


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
            self._stop.wait(0.5)

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
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_setup(n_gpus):
    import torch
    import torch.distributed as dist
    if n_gpus > 1 or "RANK" in os.environ:
        dist.init_process_group(os.environ.get("LBDD_BENCH_BACKEND", "nccl"))
        rank = dist.get_rank()
        world = dist.get_world_size()
        local = int(os.environ.get("LOCAL_RANK", rank))
        local = int(os.environ.get("LBDD_BENCH_DEVICE", local))  # tests: ranks share a GPU
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


def reduce_scalar(x: float, op: str) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return x
    t = torch.tensor([x], dtype=torch.float64,
                     device="cpu" if dist.get_backend() == "gloo" else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.MIN)
    return float(t.item())


# ---------------------------------------------------------------------------
# the reference on the host cores (oracle/_ref only; never the product .so)
# ---------------------------------------------------------------------------

def load_checkpoint():
    """The reference's own mid-solve state: centers of the first X arrivals
    in arrival order (int16, zlib), written by oracle/run_ref_scale.py."""
    meta = committed_json("ref_cpu_profile_configs1.json")
    if not meta or not meta.get("checkpoint"):
        return None, None
    import numpy as np
    path = os.path.join(CKPT_DIR, meta["checkpoint"]["file"])
    with open(path, "rb") as f:
        cs = np.frombuffer(zlib.decompress(f.read()), dtype=np.int16).copy()
    return cs, meta


def cpu_estimate(meta, first_box_s, first_n, steady_box_s_per_arrival):
    """Whole-solve CPU time on this box from two bounded samples.

    The reference's full configs[1] run in the build container
    (profiles/ref_cpu_profile_configs1.json: time marks every few thousand
    arrivals, as far as it got) gives the time profile t_here(x). On this box
    we time (1) the first `first_n` arrivals from scratch and (2) arrivals
    continued from the reference's checkpoint at X; their ratios to the same
    samples in the build container calibrate the box's speed for the early
    and the steady-state phase. Arrivals past the profile's last mark are
    extrapolated at the last measured rate (a lower bound: the rate grows as
    heaps fill and overloads spread).
    """
    if meta is None:
        return None, "no committed reference profile"
    here = meta["here"]
    speed_first = first_box_s / here["first_loop_s"]
    speed_steady = steady_box_s_per_arrival / here["steady_s_per_arrival"]
    x_ck = meta["checkpoint"]["arrivals"]
    marks = meta["marks_s"]          # cumulative loop seconds at (i+1)*mark_every arrivals
    every = meta["mark_every"]
    n = meta["n"]
    t_ck_here = meta["checkpoint"]["loop_s_here"]
    covered = len(marks) * every
    t_covered = marks[-1]
    # the last window's rate: the per-arrival cost keeps growing, so this is
    # the tightest lower bound the profile supports
    tail_rate = (marks[-1] - marks[-2]) / every if len(marks) > 1 else marks[-1] / every
    t_full_here = t_covered + tail_rate * max(0, n - covered)
    # phase 1 (0 .. X) at the early speed ratio, the rest at the steady ratio
    est = (meta["setup_s_here"] * speed_first + t_ck_here * speed_first
           + (t_full_here - t_ck_here) * speed_steady)
    note = (f"profile covers {covered} of {n} arrivals ({t_covered:.0f} s loop in the build "
            f"container); the remaining {max(0, n - covered)} extrapolated at the last rate "
            f"{tail_rate * 1e3:.1f} ms/arrival (lower bound); box/container speed "
            f"{speed_first:.2f} (first {first_n} arrivals), {speed_steady:.2f} (steady state "
            f"from checkpoint {x_ck})")
    return est, note


class RefSampler:
    """Bounded samples of the reference's asral loop on configs[1]."""

    def __init__(self, problem):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import ctypes as C
        import pyoracle
        self.C = C
        self.lib = pyoracle.reference()
        self.kind = "reference"
        if self.lib is None:
            raise RuntimeError("oracle/_ref/liblbdd_ref.so missing (build() compiles it)")
        self.inst = self.lib.instance(problem)
        self.resumed = None
        self.ck_arrivals = 0

    def first(self, arrivals):
        ns, done, setup = self.inst.sample(arrivals)
        return (ns - setup) / 1e9, setup / 1e9, done

    def open_checkpoint(self, cs):
        C = self.C
        new = self.lib._fn("resume_new")
        new.restype = C.c_void_p
        setup = C.c_int64()
        self.resumed = new(C.c_void_p(self.inst.h), cs.ctypes.data_as(C.POINTER(C.c_int16)),
                           C.c_int64(len(cs)), C.byref(setup))
        if not self.resumed:
            raise RuntimeError(self.lib._err().decode())
        self.ck_arrivals = len(cs)
        return setup.value / 1e9

    def steady(self, arrivals):
        C = self.C
        ns, done = C.c_int64(), C.c_int64()
        self.lib._check(self.lib._fn("resume_step")(C.c_void_p(self.resumed), C.c_int64(arrivals),
                                                    C.byref(ns), C.byref(done)))
        return ns.value / 1e9, done.value

    def close(self):
        if self.resumed:
            self.lib._fn("resume_free")(self.C.c_void_p(self.resumed))
            self.resumed = None
        self.inst.close()


def config0_reference():
    """configs[0] (10K x 100, 80% capacity, uniform penalties) solved to
    completion by the stock reference lbdd::asral_solve on this host."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    import synth_instances as SI
    prob = SI.problem(SI.CONFIG0)
    lib = pyoracle.reference()
    t0 = time.perf_counter()
    r = lib.solve(prob, "asral")
    el = time.perf_counter() - t0
    return {"spec": SI.CONFIG0.name(), "reference_s": round(el, 3), "objective": r.objective,
            "assignment_sha256": SI.assignment_sha256(r.assignment), "cores": 1}


def cpu_leg(problem, a, budget_s):
    """Our arm's cpu_baseline: one first-arrivals sample + one steady-state
    sample of the reference, calibrated by cpu_estimate()."""
    cs, meta = load_checkpoint()
    rs = RefSampler(problem)
    try:
        t_first, setup_s, nfirst = rs.first(a.ref_first)
        if cs is None:
            est = setup_s + t_first / max(nfirst, 1) * problem.n
            return {"value": round(est, 1), "unit": "s", "cores": 1, "kind": rs.kind,
                    "sample": f"first {nfirst} arrivals ({t_first:.1f} s), linear extrapolation "
                              "(no committed checkpoint; lower bound)"}
        rs.open_checkpoint(cs)
        t_st, nst = rs.steady(a.ref_arrivals)
        est, note = cpu_estimate(meta, t_first, nfirst, t_st / max(nst, 1))
        return {"value": round(est, 1), "unit": "s", "cores": 1, "kind": rs.kind,
                "sample": f"first {nfirst} arrivals from scratch ({t_first:.1f} s loop + "
                          f"{setup_s:.1f} s setup) and {nst} arrivals resumed from the "
                          f"reference's own checkpoint after {len(cs)} arrivals "
                          f"({t_st:.1f} s); {note}"}
    finally:
        rs.close()


def run_reference(a):
    """The reference arm: rank 0 only, the reference's CPU solver."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    t_begin = time.time()
    import synth_instances as SI
    spec, is_cfg1 = spec_of(a)
    prob = SI.problem(spec)
    sha = SI.instance_sha256(prob.costs, spec)
    cs, meta = load_checkpoint() if is_cfg1 else (None, None)
    rs = RefSampler(prob)
    cfg0 = config0_reference()
    if cs is not None:
        rs.open_checkpoint(cs)
    vals, firsts, steadies = [], [], []
    ran_w = ran_k = 0
    for step in range(a.warmup + a.steps):
        if step >= 1 and time.time() - t_begin > a.budget * 0.8:
            break
        t_first, setup_s, nfirst = rs.first(a.ref_first)
        if cs is not None:
            t_st, nst = rs.steady(a.ref_arrivals)
            est, note = cpu_estimate(meta, t_first, nfirst, t_st / max(nst, 1))
        else:
            t_st, nst = 0.0, 0
            est = setup_s + t_first / max(nfirst, 1) * spec.n
            note = "linear extrapolation of the first arrivals (lower bound)"
        if step < a.warmup:
            ran_w += 1
            continue
        ran_k += 1
        vals.append(est)
        firsts.append(t_first)
        steadies.append(t_st / max(nst, 1))
    if not vals:  # budget hit during warm-up: the last sample is the step
        vals.append(est)
        ran_k = 1
    rs.close()
    v = round(statistics.mean(vals), 1)
    line = {"impl": "reference", "metric": "asral_solve_time_s", "value": v, "unit": "s",
            "n_gpus": a.gpus, "steps": ran_k, "warmup": ran_w, "requested_steps": a.steps,
            "requested_warmup": a.warmup, "ms_per_step": round(v * 1e3, 1),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (synth_instances.py, host-generated; same bytes as the repo arm)",
            "config": {"workload": workload_name(spec, is_cfg1), "spec": spec.name(),
                       "n_demands": spec.n, "n_centers": spec.k, "instance_sha256": sha},
            "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": rs.kind,
                             "sample": f"per step: first {a.ref_first} arrivals from scratch "
                                       f"(mean {statistics.mean(firsts):.1f} s) + "
                                       f"{a.ref_arrivals} arrivals resumed from the reference's "
                                       f"checkpoint (mean {statistics.mean(steadies) * 1e3:.0f} "
                                       f"ms/arrival); {note}; sequential stock loop "
                                       "(para-ASRAL's worker pool can lose a wake-up, DESIGN.md §6)"},
            "config0": cfg0,
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "native_libs": "oracle/_ref/liblbdd_ref.so only",
            "wall_s": round(time.time() - t_begin, 1)}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_sharded(a):
    """N > 1: the configs[1] matrix split in row blocks over the ranks
    (sharded.ShardedInstance: CUDA IPC row table, per-block arrival scans
    all-gathered over NCCL, replicated arrival loop). One step = one solve
    on every rank; value = the max over ranks of the device time."""
    t_begin = time.time()
    import torch
    import torch.distributed as dist

    import synth_instances as SI
    from paper_2304_06543_b200 import solver as S
    from paper_2304_06543_b200.sharded import ShardedInstance, block_range

    rank, world, local = dist_setup(a.gpus)
    spec, is_cfg1 = spec_of(a)
    n, k = spec.n, spec.k
    row0, rows = block_range(n, world, rank)
    host = SI.cost_rows(spec, row0, rows)          # this rank's rows only
    inst = ShardedInstance(host, n, SI.centers(spec), device=local)
    t_ready = time.time()
    warm_s = []
    while len(warm_s) < max(1, a.warmup):
        if warm_s and time.time() - t_begin > 0.3 * a.budget:
            break
        r = inst.solve("asral", want_assignment=False)
        warm_s.append(r.timings.device_ns / 1e9)
    barrier()
    per_solve = reduce_scalar(max(warm_s), "max") * 1.05 + 1.0
    fit = int((a.budget - (time.time() - t_begin) - per_solve - 60) // per_solve)
    steps = int(reduce_scalar(float(max(1, min(a.steps, fit))), "min"))
    launches0 = S.launch_count()
    reports = []
    with ClockSampler(local) as clocks:
        for _ in range(steps):
            barrier()
            reports.append(inst.solve("asral", want_assignment=False))
        barrier()
    launches = S.launch_count() - launches0
    step_s = reduce_scalar(statistics.mean(r.timings.device_ns / 1e9 for r in reports), "max")
    rep = reports[-1]
    # e2e: this rank's block from host memory, the solve, the assignment back
    barrier()
    t0 = time.perf_counter()
    inst.close()
    inst = ShardedInstance(host, n, SI.centers(spec), device=local)
    r2 = inst.solve("asral", want_assignment=True)
    e2e_s = reduce_scalar(time.perf_counter() - t0, "max")
    assert r2.objective == rep.objective
    line = {
        "metric": "asral_solve_time_s", "baseline_metric": BASELINE_METRIC,
        "value": round(step_s, 4), "unit": "s", "n_gpus": world, "steps": steps,
        "warmup": len(warm_s), "requested_steps": a.steps, "requested_warmup": a.warmup,
        "ms_per_step": round(step_s * 1e3, 2), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (synth_instances.py lbdd-synth-v2, host-generated per row block)",
        "config": {"workload": workload_name(spec, is_cfg1), "spec": spec.name(),
                   "n_demands": n, "n_centers": k,
                   "parallelism": f"rows sharded over {world} GPUs (CUDA IPC row table, "
                                  "per-block arrival scans all-gathered over NCCL); the "
                                  "sequential arrival loop replicated on every rank",
                   "rows_per_rank": block_range(n, world, 0)[1],
                   "l2": "inputs larger than L2; no flush needed",
                   "objective": rep.objective,
                   "assignment_sha256": SI.assignment_sha256(r2.assignment)},
        "e2e": {"value": round(e2e_s, 4), "unit": "s",
                "h2d_bytes_per_step": int(rows * k * 4), "d2h_bytes_per_step": int(n * 4),
                "path": "per rank: block upload from host + IPC exchange + sharded solve + "
                        "assignment to host"},
        "gpu_launches": int(launches // max(steps, 1)),
        "roofline": {"kernel": "cluster_engine_kernel", "bound": "hbm",
                     "achieved": round((n + rep.stats.transfers_applied) * k * 4
                                       / max(rep.timings.engine_ns, 1), 3),
                     "peak": peaks()[0], "unit": "GB/s",
                     "frac": round((n + rep.stats.transfers_applied) * k * 4
                                   / max(rep.timings.engine_ns, 1) / peaks()[0], 7),
                     "traffic": None,
                     "note": "replicated arrival loop; rows of other ranks' blocks read over "
                             "NVLink through the IPC row table"},
        "clocks": clocks.summary(), "setup_s": round(t_ready - t_begin, 1),
    }
    line["wall_s"] = round(time.time() - t_begin, 1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    inst.close()
    dist.barrier()
    dist.destroy_process_group()


def run_ours(a):
    t_begin = time.time()
    import ctypes as C

    import numpy as np
    import torch
    import torch.distributed as dist

    import synth_instances as SI
    from paper_2304_06543_b200 import _abi
    from paper_2304_06543_b200 import solver as S
    from paper_2304_06543_b200.sharded import combine_min_transfer, shard_rows

    rank, world, local = dist_setup(a.gpus)
    spec, is_cfg1 = spec_of(a)
    n, k = spec.n, spec.k

    # ---- the instance, generated on the host into pinned memory ----
    pinned = torch.empty((n, k), dtype=torch.int32).pin_memory()
    host = pinned.numpy()
    SI.costs(spec, out=host)
    cap, fam, off, par = SI.centers(spec)
    sha = SI.instance_sha256(host, spec) if rank == 0 else None
    desc = _abi.InstanceDesc(n, k, C.cast(pinned.data_ptr(), _abi.I32P),
                             cap.ctypes.data_as(_abi.I64P), fam.ctypes.data_as(_abi.I32P),
                             off.ctypes.data_as(_abi.I64P), par.ctypes.data_as(_abi.I64P))
    h = C.c_void_p()
    S._check(S._lib.lbdd_b200_instance_create(C.byref(desc), local, C.byref(h)))
    dev = S.DeviceInstance(h.value)
    t_ready = time.time()

    # ---- warm-up solves (at least one), then as many timed solves as fit ----
    warm_s = []
    while len(warm_s) < max(1, a.warmup):
        if warm_s and time.time() - t_begin > 0.3 * a.budget:
            break
        r = S.asral_solve(dev, want_assignment=False)
        warm_s.append(r.timings.device_ns / 1e9)
    barrier()
    per_solve = reduce_scalar(max(warm_s), "max") * 1.05 + 0.5
    reserve = per_solve + 25.0 + (90.0 if (rank == 0 and world == 1) else 0.0) + 30.0
    fit = int((a.budget - (time.time() - t_begin) - reserve) // per_solve)
    steps = int(reduce_scalar(float(max(1, min(a.steps, fit))), "min"))
    launches0 = S.launch_count()
    reports = []
    with ClockSampler(local) as clocks:
        t0 = time.perf_counter()
        for _ in range(steps):
            reports.append(S.asral_solve(dev, want_assignment=False))
        barrier()
        wall = time.perf_counter() - t0
    launches = S.launch_count() - launches0
    # device time: CUDA events recorded by the library on the stream it
    # launches on, around each whole solve (report.timings.device_ns)
    dev_s = [r.timings.device_ns / 1e9 for r in reports]
    step_s = reduce_scalar(statistics.mean(dev_s), "max")
    rep = reports[-1]
    objective = rep.objective
    assert all(r.objective == objective for r in reports), "solves disagree"

    # ---- e2e through the C ABI with host buffers (one solve) ----
    assign_host = torch.empty(n, dtype=torch.int32).pin_memory()
    load_host = np.zeros(k + 1, np.int64)
    barrier()
    t0 = time.perf_counter()
    h2 = C.c_void_p()
    S._check(S._lib.lbdd_b200_instance_create(C.byref(desc), local, C.byref(h2)))
    oc, keep = S.SolverOptions().to_c()
    r2 = _abi.SolveReportC()
    S._check(S._lib.lbdd_b200_solve(h2, 0, C.byref(oc), C.byref(r2),
                                    C.cast(assign_host.data_ptr(), _abi.I32P),
                                    load_host.ctypes.data_as(_abi.I64P)))
    S._check(S._lib.lbdd_b200_instance_destroy(h2))
    e2e_s = reduce_scalar(time.perf_counter() - t0, "max")
    assert r2.objective == objective, "e2e objective differs from the resident solve"
    assignment_sha = SI.assignment_sha256(assign_host.numpy())

    # ---- the full-matrix scan (build_index), single and sharded ----
    bc, _, _ = S.arrival_queue(dev)
    ms, nbytes = S.bench_index_scan(dev, 5)
    scan_gbs = nbytes / (ms / 1e3) / 1e9
    row0, rows = shard_rows(n, world, rank)
    d_assign = torch.from_numpy(bc).cuda()
    part = torch.empty(k * k, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(2):
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
    shard_ms = reduce_scalar(e0.elapsed_time(e1) / 5, "max")
    sharded_ok = None
    if world > 1 and rank == 0:
        full = torch.from_numpy(S.build_index(dev, bc).reshape(-1)).cuda()
        sharded_ok = bool(torch.equal(full, part))

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
    barriers = rep.timings.grid_barriers
    us_per_barrier = rep.timings.engine_ns / 1e3 / max(barriers, 1)
    lat = committed_json("cluster_latency.json") or {}
    floor_us = lat.get("barrier_exchange_us")
    traffic = committed_json("engine_traffic.json") or {}
    line = {
        "metric": "asral_solve_time_s",
        "baseline_metric": BASELINE_METRIC,
        "value": round(step_s, 4),
        "unit": "s",
        "n_gpus": world,
        "steps": steps,
        "warmup": len(warm_s),
        "requested_steps": a.steps,
        "requested_warmup": a.warmup,
        "ms_per_step": round(step_s * 1e3, 2),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic (synth_instances.py lbdd-synth-v2, host-generated, uploaded)",
        "config": {"workload": workload_name(spec, is_cfg1), "spec": spec.name(),
                   "n_demands": n, "n_centers": k, "instance_sha256": sha,
                   "parallelism": f"replicas x{world} (solve), rows sharded x{world} (scan)",
                   "l2": "inputs (4 GB cost matrix) larger than L2 (126 MB); no flush needed",
                   "objective": objective, "assignment_sha256": assignment_sha},
        "e2e": {"value": round(e2e_s, 4), "unit": "s",
                "h2d_bytes_per_step": int(n * k * 4 + cap.nbytes + fam.nbytes + off.nbytes
                                          + par.nbytes),
                "d2h_bytes_per_step": int(n * 4 + load_host.nbytes),
                "path": "lbdd_b200_instance_create (pinned host) + lbdd_b200_solve + assignment "
                        "to pinned host + lbdd_b200_instance_destroy"},
        "gpu_launches": int(launches // max(steps, 1)),
        "roofline": {"kernel": "cluster_engine_kernel", "bound": "hbm",
                     "achieved": round(engine_gbs, 3), "peak": peak, "unit": "GB/s",
                     "frac": round(engine_gbs / peak, 7),
                     "traffic": traffic.get("dram_bytes_per_launch"),
                     "traffic_source": traffic.get("source"),
                     "launches_per_step": eng_launches,
                     "ms_per_launch": round(eng_ns_per_launch / 1e6, 3),
                     "share_of_step": round(rep.timings.engine_ns / max(rep.timings.device_ns, 1), 4),
                     "latency": {"us_per_barrier": round(us_per_barrier, 3),
                                 "barriers_per_arrival": round(barriers / n, 2),
                                 "floor_us_per_barrier": floor_us,
                                 "frac_of_latency_floor": (round(floor_us / us_per_barrier, 3)
                                                           if floor_us else None),
                                 "floor_source": lat.get("source")},
                     "note": f"peak {peak_kind}; the engine is latency-bound (cluster barrier "
                             "per relaxation round): judge it by latency.*; bytes = 4k per "
                             "arrival + 4k per applied transfer"},
        "scan": {"kernel": "seg_argmin_kernel (build_index full-matrix scan, incl. bucketing)",
                 "ms": round(ms, 4), "achieved": round(scan_gbs, 1), "peak": peak, "unit": "GB/s",
                 "frac": round(scan_gbs / peak, 4), "bytes": nbytes,
                 "sharded_ms_incl_allreduce": round(shard_ms, 4), "sharded_ranks": world,
                 "sharded_equals_full": sharded_ok},
        "arrival_scan": {"kernel": "row_argmin_kernel", "ms": round(rep.timings.row_scan_ns / 1e6, 4),
                         "achieved": round(row_gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(row_gbs / peak, 4), "bytes": n * k * 4},
        "host_wall_s_per_step": round(wall / steps, 4),
        "stats": {"cycle_refines": rep.stats.cycle_refine_calls,
                  "path_refines": rep.stats.path_refine_calls,
                  "cycles_removed": rep.stats.negative_cycles_removed,
                  "paths_removed": rep.stats.negative_paths_removed,
                  "transfers": rep.stats.transfers_applied,
                  "relax_rounds": rep.timings.relax_rounds, "barriers": barriers},
        "clocks": clocks.summary(),
        "setup_s": round(t_ready - t_begin, 1),
    }
    if rank == 0 and world == 1:
        try:
            line["config0"] = config0_ours(S, SI)
            line["config0"].update(config0_reference())
            line["config0"]["match"] = (line["config0"]["objective"]
                                        == line["config0"].pop("ours_objective"))
        except Exception as e:  # keep the GPU line even if the host leg fails
            line["config0"] = {"failed": repr(e)}
        try:
            from paper_2304_06543_b200.instance import ProblemInstance
            params = [list(par[off[i]:off[i + 1]]) for i in range(k)]
            problem = ProblemInstance.from_arrays(host, cap, fam, params)
            line["cpu_baseline"] = cpu_leg(problem, a, 60.0) if is_cfg1 else None
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "unit": "s", "cores": 1, "kind": "reference",
                                    "sample": f"failed: {e!r}"}
    line["wall_s"] = round(time.time() - t_begin, 1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    dev.close()
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def config0_ours(S, SI):
    """configs[0] on the GPU (device time of one solve after one warm-up)."""
    prob = SI.problem(SI.CONFIG0)
    d = S.DeviceInstance.upload(prob)
    S.asral_solve(d)
    r = S.asral_solve(d)
    d.close()
    return {"ours_s": round(r.timings.device_ns / 1e9, 4), "ours_objective": r.objective,
            "ours_assignment_sha256": SI.assignment_sha256(r.assignment)}


if __name__ == "__main__":
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 or int(os.environ.get("WORLD_SIZE", "1")) > 1:
        run_sharded(args)
    else:
        run_ours(args)
