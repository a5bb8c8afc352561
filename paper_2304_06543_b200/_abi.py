"""ctypes mirrors of the plain-C structs in include/lbdd_b200.h.

Pure struct definitions — importing this module loads no shared library.
"""
from __future__ import annotations

import ctypes as C

LBDD_OK = 0
LBDD_ERR_INVALID_ARGUMENT = 1
LBDD_ERR_LOGIC = 2
LBDD_ERR_OVERFLOW = 3
LBDD_ERR_RUNTIME = 4
LBDD_ERR_CUDA = 5

PENALTY_CONSTANT = 0
PENALTY_LINEAR = 1
PENALTY_TABLE = 2

SOLVER_ASRAL = 0
SOLVER_PARA_ASRAL = 1
SOLVER_STRICT = 2
SOLVER_GREEDY = 3

SOLVER_IDS = {"asral": SOLVER_ASRAL, "para-asral": SOLVER_PARA_ASRAL,
              "strict": SOLVER_STRICT, "greedy": SOLVER_GREEDY}
SOLVER_NAMES = {v: k for k, v in SOLVER_IDS.items()}

I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)


class InstanceDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("k", C.c_int64),
        ("costs", I32P),
        ("capacity", I64P),
        ("penalty_family", I32P),
        ("penalty_offset", I64P),
        ("penalty_params", I64P),
    ]


class SolverOptionsC(C.Structure):
    _fields_ = [
        ("parallel", C.c_int32),
        ("check_invariants", C.c_int32),
        ("refine_to_fixpoint", C.c_int32),
        ("workers", C.c_int32),
        ("chunking", C.c_int64),
        ("relax_phase", C.c_int32),
        ("index_update_phase", C.c_int32),
        ("strict_order", I32P),
        ("strict_order_len", C.c_int64),
    ]


class SolveReportC(C.Structure):
    _fields_ = [
        ("objective", C.c_int64),
        ("strict_surcharge", C.c_int64),
        ("has_dummy_center", C.c_int32),
        ("solver", C.c_int32),
        ("cycle_refine_calls", C.c_int64),
        ("path_refine_calls", C.c_int64),
        ("negative_cycles_removed", C.c_int64),
        ("negative_paths_removed", C.c_int64),
        ("refinement_gain", C.c_int64),
        ("transfers_applied", C.c_int64),
        ("invariant_checks", C.c_int64),
        ("index_update_ns", C.c_int64),
        ("bellman_ford_ns", C.c_int64),
        ("total_ns", C.c_int64),
        ("scan_ns", C.c_int64),
        ("relax_rounds", C.c_int64),
        ("grid_barriers", C.c_int64),
        ("device_ns", C.c_int64),
        ("engine_ns", C.c_int64),
        ("engine_launches", C.c_int64),
        ("row_scan_ns", C.c_int64),
    ]


class LbddError(RuntimeError):
    """Base class; the concrete class mirrors the reference's exception."""


class LbddInvalidArgument(LbddError, ValueError):
    """std::invalid_argument in the reference."""


class LbddLogicError(LbddError):
    """std::logic_error in the reference."""


class LbddOverflowError(LbddError, OverflowError):
    """std::overflow_error in the reference."""


class LbddRuntimeError(LbddError):
    """std::runtime_error in the reference."""


class LbddCudaError(LbddError):
    """Device failure."""


_ERRORS = {
    LBDD_ERR_INVALID_ARGUMENT: LbddInvalidArgument,
    LBDD_ERR_LOGIC: LbddLogicError,
    LBDD_ERR_OVERFLOW: LbddOverflowError,
    LBDD_ERR_RUNTIME: LbddRuntimeError,
    LBDD_ERR_CUDA: LbddCudaError,
}


def raise_for(code: int, message: str) -> None:
    if code == LBDD_OK:
        return
    raise _ERRORS.get(code, LbddError)(message)
