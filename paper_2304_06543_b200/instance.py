"""Host-side mirror of the reference's domain types (core.hpp).

ProblemInstance / ServiceCenter / PenaltySpec / SolverOptions / SolveReport
keep the reference's names and meaning (/root/reference/proj/include/lbdd/
core.hpp:43-143, 316-368; solver.hpp:22-32). Costs are held as an (n, k)
int32 numpy array — the device path's arithmetic type.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi

K_UNASSIGNED = -1  # core.hpp:21


@dataclass
class PenaltySpec:
    """PenaltySpec, core.hpp:43-96: q(j) for the j-th overload."""

    family: int = _abi.PENALTY_CONSTANT
    params: List[int] = field(default_factory=lambda: [1])

    @staticmethod
    def constant(p: int) -> "PenaltySpec":
        return PenaltySpec(_abi.PENALTY_CONSTANT, [int(p)])

    @staticmethod
    def linear(base: int, step: int) -> "PenaltySpec":
        return PenaltySpec(_abi.PENALTY_LINEAR, [int(base), int(step)])

    @staticmethod
    def table(values: Sequence[int]) -> "PenaltySpec":
        return PenaltySpec(_abi.PENALTY_TABLE, [int(v) for v in values])

    def at(self, j: int) -> int:
        """core.hpp:60-74."""
        if j < 1:
            raise _abi.LbddLogicError("lbdd: penalty index must be >= 1")
        if self.family == _abi.PENALTY_CONSTANT:
            return self.params[0]
        if self.family == _abi.PENALTY_LINEAR:
            return self.params[0] + self.params[1] * (j - 1)
        return self.params[min(j, len(self.params)) - 1]

    def total(self, m: int) -> int:
        """core.hpp:77-95."""
        if m <= 0:
            return 0
        if self.family == _abi.PENALTY_CONSTANT:
            return self.params[0] * m
        if self.family == _abi.PENALTY_LINEAR:
            return self.params[0] * m + self.params[1] * (m * (m - 1) // 2)
        return sum(self.at(j) for j in range(1, m + 1))


@dataclass
class ServiceCenter:
    """ServiceCenter, core.hpp:98-102."""

    id: int
    capacity: int
    penalty: PenaltySpec


class ProblemInstance:
    """ProblemInstance, core.hpp:130-143 (costs: (n, k) int32 array)."""

    def __init__(self, centers: List[ServiceCenter], costs: np.ndarray):
        costs = np.asarray(costs)
        if costs.ndim != 2:
            raise _abi.LbddInvalidArgument("lbdd: cost matrix size mismatch")
        if costs.size and (costs.max() > np.iinfo(np.int32).max):
            raise _abi.LbddInvalidArgument(
                "lbdd_b200: cost exceeds the device int32 range")
        self.centers = centers
        self.costs = np.ascontiguousarray(costs, dtype=np.int32)

    @property
    def n(self) -> int:
        return int(self.costs.shape[0])

    @property
    def k(self) -> int:
        return len(self.centers)

    def total_capacity(self) -> int:
        return sum(c.capacity for c in self.centers)

    @staticmethod
    def from_arrays(costs, capacity, penalty_family, penalty_params) -> "ProblemInstance":
        centers = [ServiceCenter(i, int(capacity[i]),
                                 PenaltySpec(int(penalty_family[i]), [int(x) for x in penalty_params[i]]))
                   for i in range(len(capacity))]
        return ProblemInstance(centers, costs)

    def desc(self) -> "DescHolder":
        return DescHolder(self)


class DescHolder:
    """Owns the numpy buffers behind an lbdd_instance_desc."""

    def __init__(self, inst: ProblemInstance):
        k = inst.k
        self.costs = inst.costs
        self.capacity = np.array([c.capacity for c in inst.centers], dtype=np.int64)
        self.family = np.array([c.penalty.family for c in inst.centers], dtype=np.int32)
        lens = [len(c.penalty.params) for c in inst.centers]
        self.offset = np.zeros(k + 1, dtype=np.int64)
        self.offset[1:] = np.cumsum(lens)
        flat = [p for c in inst.centers for p in c.penalty.params]
        self.params = np.array(flat if flat else [0], dtype=np.int64)
        self.c = _abi.InstanceDesc(
            inst.n, k,
            self.costs.ctypes.data_as(_abi.I32P),
            self.capacity.ctypes.data_as(_abi.I64P),
            self.family.ctypes.data_as(_abi.I32P),
            self.offset.ctypes.data_as(_abi.I64P),
            self.params.ctypes.data_as(_abi.I64P),
        )

    @property
    def ref(self):
        return C.byref(self.c)


@dataclass
class SolverOptions:
    """SolverOptions + ParallelConfig, solver.hpp:22-32, parallel.hpp:21-27."""

    parallel: bool = False
    check_invariants: bool = False
    refine_to_fixpoint: bool = False
    workers: int = 1
    chunking: int = 256
    relax_phase: bool = True
    index_update_phase: bool = True
    strict_order: Optional[Sequence[int]] = None

    def to_c(self):
        order = None
        if self.strict_order is not None and len(self.strict_order) > 0:
            order = np.ascontiguousarray(self.strict_order, dtype=np.int32)
        c = _abi.SolverOptionsC(
            int(self.parallel), int(self.check_invariants), int(self.refine_to_fixpoint),
            int(self.workers), int(self.chunking), int(self.relax_phase),
            int(self.index_update_phase),
            order.ctypes.data_as(_abi.I32P) if order is not None else None,
            len(order) if order is not None else 0)
        return c, order  # keep `order` alive alongside the struct


@dataclass
class SolveStats:
    """SolveStats, core.hpp:316-324."""

    cycle_refine_calls: int = 0
    path_refine_calls: int = 0
    negative_cycles_removed: int = 0
    negative_paths_removed: int = 0
    refinement_gain: int = 0
    transfers_applied: int = 0
    invariant_checks: int = 0


@dataclass
class PhaseTimings:
    """PhaseTimings, core.hpp:328-337 (plus device-only scan/rounds)."""

    index_update_ns: int = 0
    bellman_ford_ns: int = 0
    total_ns: int = 0
    scan_ns: int = 0
    relax_rounds: int = 0
    grid_barriers: int = 0
    device_ns: int = 0
    engine_ns: int = 0
    engine_launches: int = 0
    row_scan_ns: int = 0

    def other_ns(self) -> int:
        return max(0, self.total_ns - self.index_update_ns - self.bellman_ford_ns)


@dataclass
class SolveReport:
    """SolveReport, core.hpp:357-368."""

    solver: str
    objective: int
    assignment: np.ndarray
    load: np.ndarray
    stats: SolveStats
    timings: PhaseTimings
    strict_surcharge: int = 0
    has_dummy_center: bool = False

    @staticmethod
    def from_c(rep: "_abi.SolveReportC", assignment, load) -> "SolveReport":
        stats = SolveStats(rep.cycle_refine_calls, rep.path_refine_calls,
                           rep.negative_cycles_removed, rep.negative_paths_removed,
                           rep.refinement_gain, rep.transfers_applied, rep.invariant_checks)
        tim = PhaseTimings(rep.index_update_ns, rep.bellman_ford_ns, rep.total_ns,
                           rep.scan_ns, rep.relax_rounds, rep.grid_barriers,
                           rep.device_ns, rep.engine_ns, rep.engine_launches,
                           rep.row_scan_ns)
        return SolveReport(_abi.SOLVER_NAMES.get(rep.solver, "?"), rep.objective, assignment,
                           load, stats, tim, rep.strict_surcharge, bool(rep.has_dummy_center))
