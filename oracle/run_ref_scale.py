"""TEST INFRASTRUCTURE ONLY — pin the GPU solve at scale with the reference.

Runs the UNMODIFIED reference's asral loop (oracle/_ref/liblbdd_ref.so,
`lbdd_ref_asral_run` = solver.hpp:133-170 closed by the reference's own
finish_report) to completion on a synth_instances.py instance and writes
tests/golden/scale/<tag>.json: the spec, objective, assignment/load sha256,
stats, and the CPU time with progress marks. Runs in the build container
(hours at configs[1]); the GPU tests regenerate the instance from the spec
and compare bit for bit.

    python oracle/run_ref_scale.py --tag k1000_n100k --n 100000 --k 1000
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import synth_instances as SI  # noqa: E402
from paper_2304_06543_b200 import _abi  # noqa: E402
from paper_2304_06543_b200.instance import DescHolder  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--tag", required=True)
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--k", type=int, required=True)
    p.add_argument("--seed", type=int, default=20250)
    p.add_argument("--theta", default="8/10")
    p.add_argument("--mark", type=int, default=10000)
    p.add_argument("--ckpt", type=int, default=0,
                   help="write resumable checkpoints every N arrivals (bench CPU samples)")
    p.add_argument("--ckpt-prefix", default="/root/refruns/ckpt_")
    a = p.parse_args()
    tn, td = (int(x) for x in a.theta.split("/"))
    spec = SI.SynthSpec(a.n, a.k, seed=a.seed, theta_num=tn, theta_den=td)
    t0 = time.time()
    prob = SI.problem(spec)
    sha = SI.instance_sha256(prob.costs, spec)
    print(f"generated {spec.name()} in {time.time() - t0:.1f} s sha {sha}", flush=True)
    lib = C.CDLL(os.path.join(HERE, "_ref", "liblbdd_ref.so"))
    lib.lbdd_ref_last_error.restype = C.c_char_p
    h = DescHolder(prob)
    nmarks = a.n // a.mark + 1
    marks = np.zeros(nmarks, np.int64)
    rep = _abi.SolveReportC()
    assign = np.full(a.n, -1, np.int32)
    load = np.zeros(a.k + 1, np.int64)
    setup = C.c_int64()
    t0 = time.time()
    rc = lib.lbdd_ref_asral_run(h.ref, C.c_int64(a.mark), marks.ctypes.data_as(_abi.I64P),
                                C.c_int64(nmarks), C.byref(rep), assign.ctypes.data_as(_abi.I32P),
                                load.ctypes.data_as(_abi.I64P), C.byref(setup),
                                C.c_int64(a.ckpt), a.ckpt_prefix.encode())
    wall = time.time() - t0
    if rc != 0:
        raise SystemExit(f"reference failed rc={rc}: {lib.lbdd_ref_last_error().decode()}")
    out = {
        "spec": spec.__dict__, "spec_name": spec.name(), "instance_sha256": sha,
        "solver": "asral (reference, sequential)",
        "objective": rep.objective,
        "assignment_sha256": SI.assignment_sha256(assign),
        "load": load[:a.k].tolist(),
        "stats": {f: getattr(rep, f) for f in ("cycle_refine_calls", "path_refine_calls",
                                               "negative_cycles_removed", "negative_paths_removed",
                                               "refinement_gain", "transfers_applied")},
        "cpu_seconds": round(wall, 2), "setup_seconds": round(setup.value / 1e9, 2),
        "cores": 1, "host": os.uname().nodename, "cpu": _cpu_model(),
        "mark_every": a.mark, "marks_s": [round(m / 1e9, 2) for m in marks if m > 0],
        "made_by": "oracle/run_ref_scale.py (oracle/_ref/liblbdd_ref.so, -O3 -DNDEBUG)",
    }
    path = os.path.join(ROOT, "tests", "golden", "scale", a.tag + ".json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {path}: objective {rep.objective} in {wall:.1f} s", flush=True)


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "?"


if __name__ == "__main__":
    main()
