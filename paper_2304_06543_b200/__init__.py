"""B200-native ASRAL solver for Load Balanced Demand Distribution.

Host side mirrors the reference's C++ API (lbdd::asral_solve / strict_solve /
greedy_solve / build_index ...); the hot path runs in hand-written sm_100a
CUDA kernels behind the C ABI in include/lbdd_b200.h (lib/liblbdd_b200.so).
"""
from .instance import (K_UNASSIGNED, PenaltySpec, PhaseTimings, ProblemInstance,  # noqa: F401
                       ServiceCenter, SolveReport, SolverOptions, SolveStats)
from ._abi import (LbddError, LbddInvalidArgument, LbddLogicError,  # noqa: F401
                   LbddOverflowError, LbddRuntimeError, LbddCudaError)

__version__ = "0.1.0"


def __getattr__(name):
    # solver entry points load the CUDA library on first use (and fail loudly
    # when it is missing) — importing the package itself stays cheap.
    if name.startswith("__"):
        raise AttributeError(name)
    import importlib
    solver = importlib.import_module(__name__ + ".solver")
    if name == "solver":
        return solver
    if hasattr(solver, name):
        return getattr(solver, name)
    raise AttributeError(name)
