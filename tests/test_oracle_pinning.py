"""The oracle (oracle/liblbdd_oracle.c) pinned against the reference.

* against the reference tests' known answers (solver_test.cpp,
  refine_test.cpp, subspace_test.cpp, instgen_test.cpp) — restated here;
* against golden fixtures produced by the UNMODIFIED reference
  (tests/golden/make_golden.py);
* against the compiled reference itself (oracle/_ref) when it is present.
"""
import hashlib

import numpy as np
import pytest

from conftest import instance_from_json, load_golden
import pyoracle as po
from paper_2304_06543_b200.instance import PenaltySpec, ProblemInstance, ServiceCenter, SolverOptions
from paper_2304_06543_b200 import LbddInvalidArgument, LbddLogicError


def column_instance(column, capacity, penalty):
    return ProblemInstance([ServiceCenter(0, capacity, PenaltySpec.constant(penalty))],
                           np.array(column, np.int32).reshape(-1, 1))


def worked_cycle_instance():  # refine_test.cpp:99-111
    return ProblemInstance([ServiceCenter(s, 2, PenaltySpec.constant(5)) for s in range(4)],
                           np.array([[10, 6, 20, 20], [20, 10, 7, 20], [20, 20, 10, 7],
                                     [7, 20, 20, 10]], np.int32))


def worked_path_instance():  # refine_test.cpp:145-159
    cs = [ServiceCenter(0, 1, PenaltySpec.constant(20)), ServiceCenter(1, 1, PenaltySpec.constant(100)),
          ServiceCenter(2, 1, PenaltySpec.constant(100)), ServiceCenter(3, 2, PenaltySpec.constant(100))]
    return ProblemInstance(cs, np.array([[10, 5, 20, 20], [30, 10, 6, 30], [30, 30, 10, 6],
                                         [25, 25, 25, 10], [10, 30, 30, 30]], np.int32))


# ---- known answers from the reference's own tests ----

def test_single_demand(oracle):  # solver_test.cpp:25
    r = oracle.solve(column_instance([4], 1, 10), "asral")
    assert r.objective == 4 and r.assignment[0] == 0


def test_forced_overload(oracle):  # solver_test.cpp:32
    r = oracle.solve(column_instance([4, 6], 1, 10), "asral")
    assert r.objective == 20
    assert r.stats.negative_cycles_removed == 0 and r.stats.negative_paths_removed == 0


def test_rejects_invalid_instance(oracle):  # solver_test.cpp:99
    with pytest.raises(LbddInvalidArgument):
        oracle.solve(column_instance([0], 1, 10), "asral")


def test_strict_diagonal(oracle):  # solver_test.cpp:120
    inst = ProblemInstance([ServiceCenter(0, 1, PenaltySpec.constant(5)),
                            ServiceCenter(1, 1, PenaltySpec.constant(5))],
                           np.array([[1, 9], [9, 1]], np.int32))
    r = oracle.solve(inst, "strict")
    assert r.objective == 2 and list(r.assignment) == [0, 1] and r.strict_surcharge == 0


def test_strict_excess_demand(oracle):  # solver_test.cpp:134
    r = oracle.solve(column_instance([2, 3, 4], 1, 10), "strict")
    assert r.objective == 2 and r.strict_surcharge == 10 and r.has_dummy_center
    assert list(r.assignment) == [0, 1, 1]


def test_worked_cycle_drops_thirteen(oracle):  # refine_test.cpp:113
    applied, gain, a, _ = oracle.refine(worked_cycle_instance(), 0, 0, [0, 1, 2, 3])
    assert applied and gain == -13
    assert oracle.evaluate_objective(worked_cycle_instance(), a) == 27


def test_worked_path_drops_thirtythree(oracle):  # refine_test.cpp:161
    inst = worked_path_instance()
    applied, gain, a, _ = oracle.refine(inst, 1, 0, [0, 1, 2, 3, 0])
    assert applied and gain == -33
    assert oracle.evaluate_objective(inst, a) == 70 - 33
    assert np.bincount(a, minlength=4).tolist() == [1, 1, 1, 2]


def test_free_capacity_chain_refund(oracle):  # refine_test.cpp:184
    inst = ProblemInstance([ServiceCenter(0, 0, PenaltySpec.constant(10)),
                            ServiceCenter(1, 1, PenaltySpec.constant(7))],
                           np.array([[4, 4]], np.int32))
    applied, gain, _, _ = oracle.refine(inst, 1, 0, [0])
    assert applied and gain == -10


def test_path_refine_requires_overload(oracle):  # refine_test.cpp:201
    with pytest.raises(LbddLogicError):
        oracle.refine(worked_cycle_instance(), 1, 0, [0, -1, -1, -1])


def test_negative_cycle_witness(oracle):  # refine_test.cpp:85
    w = np.full((3, 4), po.NO_EDGE, np.int64)
    w[0, 1], w[1, 2], w[2, 1], w[2, 3] = 0, -5, -5, 0
    with pytest.raises(LbddLogicError):
        oracle.lowest_cost_path(w, 0)


def test_single_edge_path(oracle):  # refine_test.cpp:42
    w = np.full((1, 2), po.NO_EDGE, np.int64)
    w[0, 1] = -13
    cost, dist, par, path = oracle.lowest_cost_path(w, 0)
    assert cost == -13 and list(path) == [0, 1] and par[1] == 0


def test_unreachable_sink(oracle):  # refine_test.cpp:55
    w = np.full((2, 3), po.NO_EDGE, np.int64)
    w[0, 1] = 5
    assert oracle.lowest_cost_path(w, 0) is None


def test_build_index_known(oracle):  # subspace_test.cpp:50, 121
    inst = ProblemInstance([ServiceCenter(i, 1, PenaltySpec.constant(1)) for i in range(2)],
                           np.array([[3, 5]], np.int32))
    m = oracle.build_index(inst, [0])
    assert m[0, 1] == (2 << 32) | 0 and m[1, 0] == po.NO_EDGE
    inst = ProblemInstance([ServiceCenter(i, 2, PenaltySpec.constant(1)) for i in range(2)],
                           np.array([[3, 5], [9, 5]], np.int32))
    m = oracle.build_index(inst, [0, 0])
    assert (m[0, 1] >> 32) == -4 and (m[0, 1] & 0xffffffff) == 1


def test_derive_center_count(oracle):  # instgen_test.cpp:41
    for n, ratio, k in [(65771, 500.0, 131), (65793, 600.0, 109), (65808, 700.0, 94),
                        (65820, 800.0, 82), (65829, 900.0, 73), (3, 10.0, 1)]:
        assert po.oracle().lib.lbdd_oracle_derive_center_count(
            po.C.c_int64(n), po.C.c_double(ratio)) == k


# ---- golden fixtures from the reference ----

def _same(rep, gold):
    return (rep.objective == gold["objective"] and rep.assignment.tolist() == gold["assignment"]
            and rep.load.tolist() == gold["load"] and rep.strict_surcharge == gold["strict_surcharge"]
            and rep.stats.__dict__ == gold["stats"])


def test_random_solves_match_reference_fixtures(oracle):
    for it, case in enumerate(load_golden("random_solves.json")):
        inst = instance_from_json(case["instance"])
        for key, gold in case["reports"].items():
            solver, _, fix = key.partition("+")
            rep = oracle.solve(inst, solver, SolverOptions(refine_to_fixpoint=bool(fix),
                                                           check_invariants=(it % 4 == 0)))
            assert _same(rep, gold), (key, rep.objective, gold["objective"])
        if "mcf_optimum" in case:  # oracle <= asral <= greedy (acceptance.cpp:161)
            assert case["mcf_optimum"] <= case["reports"]["asral"]["objective"]
            assert case["reports"]["asral"]["objective"] <= case["reports"]["greedy"]["objective"]


def test_road_graph_fixtures(oracle):
    for case in load_golden("road_graph.json"):
        inst = instance_from_json(case["instance"])
        assert _same(oracle.solve(inst, "asral"), case["asral"])
        assert _same(oracle.solve(inst, "strict"), case["strict"])


def test_config0_generator_and_solves(oracle):
    g = load_golden("config0.json")
    inst = oracle.generate(g["seed"], g["n"], g["ratio"], g["theta"], *g["pen"])
    assert hashlib.sha256(inst.costs.tobytes()).hexdigest() == g["costs_sha256"]
    assert [c.capacity for c in inst.centers] == g["capacity"]
    for solver in ["greedy", "strict", "asral"]:
        r = oracle.solve(inst, solver)
        gold = g["reports"][solver]
        assert r.objective == gold["objective"]
        assert hashlib.sha256(r.assignment.astype(np.int32).tobytes()).hexdigest() == gold["assignment_sha256"]
        assert r.stats.__dict__ == gold["stats"]


# ---- live cross-check against the compiled reference ----

def test_oracle_matches_compiled_reference(oracle, reference):
    rng = po.Mt19937_64(97)
    for it in range(80):
        n = 1 + rng() % 35
        k = 1 + rng() % 6
        inst = po.random_instance(rng, n=n, k=k, total_capacity=(rng() % (n + 1)) if it % 2 else -1)
        for solver in ["asral", "strict", "greedy"]:
            a = oracle.solve(inst, solver)
            b = reference.solve(inst, solver)
            assert a.objective == b.objective and (a.assignment == b.assignment).all()
            assert a.stats == b.stats
        asg = np.array([rng() % k for _ in range(n)], np.int32)
        assert (oracle.build_index(inst, asg) == reference.build_index(inst, asg)).all()
        assert oracle.gamma_has_negative_cycle(inst, asg) == reference.gamma_has_negative_cycle(inst, asg)


def test_relaxation_matches_compiled_reference(oracle, reference):
    rng = po.Mt19937_64(157)
    for it in range(300):
        k = 2 + rng() % 6
        w = np.full((k, k + 1), po.NO_EDGE, np.int64)
        anchor = rng() % k
        for u in range(k):
            for v in range(k):
                if u != v and rng() % 10 < 6:
                    w[u, k if v == anchor else v] = (rng() % 41) - 20
        din = np.array([po.UNREACH if rng() % 4 == 0 else (rng() % 100) - 50 for _ in range(k + 1)])
        din[anchor] = 0
        pin = np.full(k + 1, -1, np.int32)
        a = oracle.relax_round(w, din, pin)
        b = reference.relax_round(w, din, pin)
        assert a[0] == b[0] and (a[1] == b[1]).all() and (a[2] == b[2]).all()
        try:
            pa = oracle.lowest_cost_path(w, anchor)
        except LbddLogicError:
            pa = "cycle"
        try:
            pb = reference.lowest_cost_path(w, anchor)
        except LbddLogicError:
            pb = "cycle"
        if isinstance(pa, str) or pa is None:
            assert pa == pb
        else:
            assert pa[0] == pb[0] and (pa[1] == pb[1]).all() and (pa[2] == pb[2]).all()
            assert (pa[3] == pb[3]).all()
