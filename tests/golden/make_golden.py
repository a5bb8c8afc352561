"""Generate the golden fixtures from the UNMODIFIED reference.

Runs in the build container only (it needs oracle/_ref/liblbdd_ref.so, which
`make -C oracle` compiles from /root/reference/proj/include). Writes small
JSON fixtures that travel with the repo; the tests read them, never the
reference tree. Re-run: python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle as po  # noqa: E402
from paper_2304_06543_b200.instance import SolverOptions  # noqa: E402


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


def inst_json(inst):
    return {
        "n": inst.n, "k": inst.k,
        "capacity": [c.capacity for c in inst.centers],
        "family": [c.penalty.family for c in inst.centers],
        "params": [c.penalty.params for c in inst.centers],
        "costs": inst.costs.reshape(-1).tolist(),
    }


def report_json(r):
    return {
        "objective": r.objective, "assignment": r.assignment.tolist(),
        "load": r.load.tolist(), "strict_surcharge": r.strict_surcharge,
        "has_dummy_center": r.has_dummy_center, "stats": r.stats.__dict__,
    }


def main():
    R = po.reference()
    if R is None:
        raise SystemExit("oracle/_ref/liblbdd_ref.so missing: run `make -C oracle` here")

    # 1. random instances drawn like the reference's own tests
    #    (tests/test_util.hpp:206 random_instance, solver_test.cpp seeds)
    cases = []
    rng = po.Mt19937_64(2031)
    for it in range(120):
        n = 1 + rng() % 40
        k = 1 + rng() % 6
        cap = (rng() % (n + 1)) if it % 3 == 0 else (n + rng() % 5 if it % 3 == 1 else -1)
        inst = po.random_instance(rng, n=n, k=k, total_capacity=cap)
        entry = {"instance": inst_json(inst), "reports": {}}
        for solver in ["asral", "strict", "greedy"]:
            for fix in [False, True]:
                opts = SolverOptions(refine_to_fixpoint=fix, check_invariants=(it % 4 == 0))
                key = f"{solver}{'+fix' if fix else ''}"
                entry["reports"][key] = report_json(R.solve(inst, solver, opts))
        if n <= 40:
            obj, sur, dummy, _ = R.oracle_solve(inst, strict=False)
            entry["mcf_optimum"] = obj
        cases.append(entry)
    with open(os.path.join(HERE, "random_solves.json"), "w") as f:
        json.dump(cases, f)

    # 2. configs[0]: |D|=10,000 x |S|=100 (ratio 100), theta 0.8, penalties
    #    1..200, euclidean, seed 42 — full reports by digest
    inst = R.generate(42, 10000, 100.0, 0.8, 1, 200)
    cfg0 = {"seed": 42, "n": 10000, "ratio": 100.0, "theta": 0.8, "pen": [1, 200],
            "costs_sha256": digest(inst.costs), "capacity": [c.capacity for c in inst.centers],
            "penalty": [c.penalty.params[0] for c in inst.centers], "reports": {}}
    for solver in ["asral", "strict", "greedy"]:
        r = R.solve(inst, solver)
        cfg0["reports"][solver] = {
            "objective": r.objective, "assignment_sha256": digest(r.assignment),
            "load": r.load.tolist(), "strict_surcharge": r.strict_surcharge,
            "stats": r.stats.__dict__}
    with open(os.path.join(HERE, "config0.json"), "w") as f:
        json.dump(cfg0, f)

    # 3. road-graph instances (instgen.hpp random_road_graph + apsp_costs),
    #    which the oracle port does not generate: store them whole
    road = []
    for seed in [11, 12, 13]:
        inst = R.generate(seed, 60, 6.0, 0.7, 1, 200, cost_source=1)
        road.append({"instance": inst_json(inst),
                     "asral": report_json(R.solve(inst, "asral")),
                     "strict": report_json(R.solve(inst, "strict"))})
    with open(os.path.join(HERE, "road_graph.json"), "w") as f:
        json.dump(road, f)
    print("wrote", len(cases), "random cases, config0, road graphs")


if __name__ == "__main__":
    main()
