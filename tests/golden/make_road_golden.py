"""Goldens for configs[3]-shaped road-network instances (synth_instances
RoadSpec, "lbdd-road-v1"), solved by the UNMODIFIED reference
(oracle/_ref/liblbdd_ref.so) in the build container: asral (and
refine_to_fixpoint) objective, assignment sha256 and stats, plus the float
objective of the float32 road costs under that assignment. The GPU test
regenerates each instance from its spec and compares bit for bit.
    python tests/golden/make_road_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle as po  # noqa: E402
import synth_instances as SI  # noqa: E402
from paper_2304_06543_b200.instance import SolverOptions  # noqa: E402

SPECS = [SI.RoadSpec(3000, 60, seed=3, vertices=2048),
         SI.RoadSpec(8000, 100, seed=5, vertices=4096),
         SI.RoadSpec(2500, 250, seed=7, vertices=4096)]


def float_objective(spec, assignment, penalties):
    """The objective with the float32 road costs (x1000, the integer cost
    units) under `assignment`, plus the (integer) penalties."""
    f = SI.road_float_rows(spec, 0, spec.n).astype(np.float64)
    return 1000.0 * float(f[np.arange(spec.n), assignment].sum()) + float(penalties)


def main():
    R = po.reference()
    out = []
    for spec in SPECS:
        prob = SI.road_problem(spec)
        entry = {"spec": spec.__dict__, "name": spec.name(), "reports": {}}
        for tag, opts in [("asral", SolverOptions()),
                          ("asral_fixpoint", SolverOptions(refine_to_fixpoint=True))]:
            r = R.solve(prob, "asral", opts)
            ints = prob.costs.astype(np.int64)[np.arange(spec.n), r.assignment].sum()
            pen = r.objective - int(ints)
            entry["reports"][tag] = {
                "objective": r.objective, "assignment_sha256": SI.assignment_sha256(r.assignment),
                "load": r.load.tolist(), "stats": r.stats.__dict__,
                "float_objective": float_objective(spec, r.assignment, pen)}
        out.append(entry)
        print(spec.name(), {t: e["objective"] for t, e in entry["reports"].items()}, flush=True)
    with open(os.path.join(HERE, "road_v1.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
