"""TEST INFRASTRUCTURE ONLY — Python handles on the parity checkers.

* ``oracle()``    — oracle/liblbdd_oracle.so, the plain-C restatement.
* ``reference()`` — oracle/_ref/liblbdd_ref.so, the UNMODIFIED reference
  compiled from /root/reference (None when it was never built).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
reference arm import this module. Also hosts ``Mt19937_64`` and
``random_instance`` — restatements of the reference tests' instance factory
(tests/test_util.hpp:195-244) so the parity tests draw the same instances
as the reference's own tests.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from paper_2304_06543_b200 import _abi
from paper_2304_06543_b200.instance import (DescHolder, PenaltySpec, ProblemInstance,
                                            ServiceCenter, SolveReport, SolverOptions)

HERE = os.path.dirname(os.path.abspath(__file__))
UNREACH = (2**63 - 1) // 4
NO_EDGE = 2**63 - 1


class CLib:
    def __init__(self, path: str, prefix: str):
        self.path = path
        self.lib = C.CDLL(path)
        self.p = prefix
        self._err = getattr(self.lib, prefix + "last_error")
        self._err.restype = C.c_char_p

    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc):
        if rc != 0:
            _abi.raise_for(rc, self._err().decode())

    # -- solvers ---------------------------------------------------------
    def solve(self, inst: ProblemInstance, solver="asral", opts: Optional[SolverOptions] = None):
        h = DescHolder(inst)
        opts = opts or SolverOptions()
        oc, keep = opts.to_c()
        rep = _abi.SolveReportC()
        assign = np.full(inst.n, -1, dtype=np.int32)
        load = np.zeros(inst.k + 1, dtype=np.int64)
        sid = _abi.SOLVER_IDS[solver] if isinstance(solver, str) else solver
        self._check(self._fn("solve")(h.ref, C.c_int32(sid), C.byref(oc), C.byref(rep),
                                      assign.ctypes.data_as(_abi.I32P),
                                      load.ctypes.data_as(_abi.I64P)))
        del keep
        kk = inst.k + 1 if rep.has_dummy_center else inst.k
        return SolveReport.from_c(rep, assign, load[:kk])

    def build_index(self, inst: ProblemInstance, assignment) -> np.ndarray:
        h = DescHolder(inst)
        a = np.ascontiguousarray(assignment, dtype=np.int32)
        out = np.empty(inst.k * inst.k, dtype=np.int64)
        self._check(self._fn("build_index")(h.ref, a.ctypes.data_as(_abi.I32P),
                                            out.ctypes.data_as(_abi.I64P)))
        return out.reshape(inst.k, inst.k)

    def refine(self, inst, kind, anchor, assignment, dummies=None):
        h = DescHolder(inst)
        a = np.ascontiguousarray(assignment, dtype=np.int32).copy()
        dm = None if dummies is None else np.ascontiguousarray(dummies, dtype=np.int64).copy()
        applied = C.c_int32()
        gain = C.c_int64()
        self._check(self._fn("refine")(h.ref, C.c_int32(kind), C.c_int32(anchor),
                                       a.ctypes.data_as(_abi.I32P),
                                       dm.ctypes.data_as(_abi.I64P) if dm is not None else None,
                                       C.byref(applied), C.byref(gain)))
        return bool(applied.value), gain.value, a, dm

    def gamma_has_negative_cycle(self, inst, assignment, dummies=None) -> bool:
        h = DescHolder(inst)
        a = np.ascontiguousarray(assignment, dtype=np.int32)
        dm = None if dummies is None else np.ascontiguousarray(dummies, dtype=np.int64)
        out = C.c_int32()
        self._check(self._fn("gamma_has_negative_cycle")(
            h.ref, a.ctypes.data_as(_abi.I32P),
            dm.ctypes.data_as(_abi.I64P) if dm is not None else None, C.byref(out)))
        return bool(out.value)

    def lowest_cost_path(self, weights: np.ndarray, anchor: int):
        """weights: (node_count-1, node_count) int64, NO_EDGE for none."""
        w = np.ascontiguousarray(weights, dtype=np.int64)
        nodes = w.shape[1]
        found = C.c_int32()
        cost = C.c_int64()
        dist = np.zeros(nodes, dtype=np.int64)
        par = np.zeros(nodes, dtype=np.int32)
        path = np.zeros(nodes + 1, dtype=np.int32)
        plen = C.c_int32()
        self._check(self._fn("lowest_cost_path")(
            C.c_int32(nodes), C.c_int32(anchor), w.ctypes.data_as(_abi.I64P), C.byref(found),
            C.byref(cost), dist.ctypes.data_as(_abi.I64P), par.ctypes.data_as(_abi.I32P),
            path.ctypes.data_as(_abi.I32P), C.byref(plen)))
        if not found.value:
            return None
        return cost.value, dist, par, path[: plen.value + 1]

    def relax_round(self, weights, dist_in, parent_in):
        w = np.ascontiguousarray(weights, dtype=np.int64)
        nodes = w.shape[1]
        din = np.ascontiguousarray(dist_in, dtype=np.int64)
        pin = np.ascontiguousarray(parent_in, dtype=np.int32)
        dout = np.zeros(nodes, dtype=np.int64)
        pout = np.zeros(nodes, dtype=np.int32)
        ch = C.c_int32()
        self._check(self._fn("relax_round")(
            C.c_int32(nodes), w.ctypes.data_as(_abi.I64P), din.ctypes.data_as(_abi.I64P),
            pin.ctypes.data_as(_abi.I32P), dout.ctypes.data_as(_abi.I64P),
            pout.ctypes.data_as(_abi.I32P), C.byref(ch)))
        return bool(ch.value), dout, pout

    def generate(self, seed, n, ratio, theta, pen_lo=1, pen_hi=200, cost_source=0,
                 road_nodes=0, avg_degree=4.0) -> ProblemInstance:
        k = C.c_int64()
        if self.p == "lbdd_ref_":
            args = (C.c_uint64(seed), C.c_int64(n), C.c_double(ratio), C.c_double(theta),
                    C.c_int64(pen_lo), C.c_int64(pen_hi), C.c_int32(cost_source),
                    C.c_int64(road_nodes), C.c_double(avg_degree), C.byref(k))
        else:
            if cost_source != 0:
                raise NotImplementedError("oracle port generates euclidean instances only")
            args = (C.c_uint64(seed), C.c_int64(n), C.c_double(ratio), C.c_double(theta),
                    C.c_int64(pen_lo), C.c_int64(pen_hi), C.byref(k))
        self._check(self._fn("generate")(*args, None, None, None))
        kk = k.value
        cap = np.zeros(kk, dtype=np.int64)
        pen = np.zeros(kk, dtype=np.int64)
        costs = np.zeros(n * kk, dtype=np.int32)
        self._check(self._fn("generate")(*args, cap.ctypes.data_as(_abi.I64P),
                                         pen.ctypes.data_as(_abi.I64P),
                                         costs.ctypes.data_as(_abi.I32P)))
        centers = [ServiceCenter(i, int(cap[i]), PenaltySpec.constant(int(pen[i])))
                   for i in range(kk)]
        return ProblemInstance(centers, costs.reshape(n, kk))

    # oracle-port-only helpers
    def evaluate_objective(self, inst, assignment, partial=False) -> int:
        h = DescHolder(inst)
        a = np.ascontiguousarray(assignment, dtype=np.int32)
        out = C.c_int64()
        self._check(self._fn("evaluate_objective")(h.ref, a.ctypes.data_as(_abi.I32P),
                                                   C.c_int32(int(partial)), C.byref(out)))
        return out.value

    def arrival_queue(self, inst):
        h = DescHolder(inst)
        bc = np.zeros(inst.n, dtype=np.int32)
        bcost = np.zeros(inst.n, dtype=np.int64)
        order = np.zeros(inst.n, dtype=np.int32)
        self._check(self._fn("arrival_queue")(h.ref, bc.ctypes.data_as(_abi.I32P),
                                              bcost.ctypes.data_as(_abi.I64P),
                                              order.ctypes.data_as(_abi.I32P)))
        return bc, bcost, order

    def asral_sample(self, inst, max_arrivals, workers=1):
        """Time the first `max_arrivals` arrivals of asral_solve's main loop.
        Returns (elapsed ns incl. setup, arrivals done, setup ns = arrival
        queue + empty index)."""
        h = DescHolder(inst)
        ns = C.c_int64()
        done = C.c_int64()
        setup = C.c_int64()
        self._check(self._fn("asral_sample")(h.ref, C.c_int64(max_arrivals), C.c_int32(workers),
                                             C.byref(ns), C.byref(done), C.byref(setup)))
        return ns.value, done.value, setup.value

    def instance(self, inst) -> "RefInstance":
        """Reference-only: the instance converted once (int64 CostMatrix) for
        repeated bounded samples (lbdd_ref_asral_sample_inst)."""
        return RefInstance(self, inst)

    def oracle_solve(self, inst, strict, size_limit=2000):
        """Reference-only: exact min-cost-flow optimum (oracle.hpp:144)."""
        h = DescHolder(inst)
        obj = C.c_int64()
        sur = C.c_int64()
        dummy = C.c_int32()
        a = np.zeros(inst.n, dtype=np.int32)
        self._check(self._fn("oracle_solve")(h.ref, C.c_int32(int(strict)), C.c_int64(size_limit),
                                             C.byref(obj), C.byref(sur), C.byref(dummy),
                                             a.ctypes.data_as(_abi.I32P)))
        return obj.value, sur.value, bool(dummy.value), a


_ORACLE = None
_REF = None


class RefInstance:
    """A reference lbdd::ProblemInstance held by oracle/_ref (bench.py's
    reference arm and cpu_baseline leg)."""

    def __init__(self, lib: CLib, inst: ProblemInstance):
        self.lib = lib
        self.n = inst.n
        new = lib._fn("instance_new")
        new.restype = C.c_void_p
        holder = DescHolder(inst)  # keeps the numpy buffers alive across the call
        self.h = new(holder.ref)
        if not self.h:
            raise RuntimeError(lib._err().decode())

    def sample(self, max_arrivals: int):
        """(elapsed ns incl. setup, arrivals done, setup ns)."""
        ns, done, setup = C.c_int64(), C.c_int64(), C.c_int64()
        self.lib._check(self.lib._fn("asral_sample_inst")(C.c_void_p(self.h),
                                                          C.c_int64(max_arrivals), C.byref(ns),
                                                          C.byref(done), C.byref(setup)))
        return ns.value, done.value, setup.value

    def close(self):
        if self.h:
            self.lib._fn("instance_free")(C.c_void_p(self.h))
            self.h = None


def oracle() -> CLib:
    global _ORACLE
    if _ORACLE is None:
        path = os.path.join(HERE, "liblbdd_oracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        _ORACLE = CLib(path, "lbdd_oracle_")
    return _ORACLE


def reference() -> Optional[CLib]:
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "liblbdd_ref.so")
        if not os.path.exists(path):
            return None
        _REF = CLib(path, "lbdd_ref_")
    return _REF


# ---------------------------------------------------------------------------
# std::mt19937_64 and the reference tests' random_instance
# ---------------------------------------------------------------------------

class Mt19937_64:
    """std::mt19937_64 (default seed 5489 when seed is None)."""

    M64 = (1 << 64) - 1

    def __init__(self, seed=5489):
        self.mt = [0] * 312
        self.mt[0] = seed & self.M64
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & self.M64
        self.idx = 312

    def __call__(self) -> int:
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self.M64


def random_instance(rng: Mt19937_64, n=10, k=3, max_cost=50, penalty_lo=1, penalty_hi=30,
                    total_capacity=-1, mixed_penalty_families=True) -> ProblemInstance:
    """lbdd_test::random_instance, tests/test_util.hpp:206-244 (same draws)."""

    def rint(lo, hi):
        return lo + rng() % (hi - lo + 1)

    total = total_capacity if total_capacity >= 0 else rint(0, n)
    caps = [0] * k
    for _ in range(total):
        caps[rint(0, k - 1)] += 1
    centers = []
    for i in range(k):
        base = rint(penalty_lo, penalty_hi)
        fam = rint(0, 2) if mixed_penalty_families else 0
        if fam == 0:
            pen = PenaltySpec.constant(base)
        elif fam == 1:
            pen = PenaltySpec.linear(base, rint(0, 5))
        else:
            table = [base]
            for _ in range(3):
                table.append(table[-1] + rint(0, 7))
            pen = PenaltySpec.table(table)
        centers.append(ServiceCenter(i, caps[i], pen))
    costs = np.array([rint(1, max_cost) for _ in range(n * k)], dtype=np.int32).reshape(n, k)
    return ProblemInstance(centers, costs)
