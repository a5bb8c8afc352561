"""Python mirror of the reference's solver API over the C ABI.

Same names and argument meaning as /root/reference/proj/include/lbdd/
solver.hpp (asral_solve, strict_solve, greedy_solve), subspace.hpp
(build_index), refine.hpp (lowest_cost_path, negative_cycle_refine,
negative_path_refine, gamma_has_negative_cycle), parallel.hpp
(parallel_relax_round) and core.hpp (evaluate_objective). Errors raise the
exception class that mirrors the reference's (see _abi.py).

Every call runs on the B200 through lib/liblbdd_b200.so. There is no CPU
fallback: if the library is missing, importing this module fails.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence, Union

import numpy as np

from . import _abi
from .instance import DescHolder, ProblemInstance, SolveReport, SolverOptions

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LBDD_B200_LIB") or os.path.join(_HERE, "lib", "liblbdd_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C paper_2304_06543_b200/csrc` "
        "(or __graft_entry__.build()); there is no CPU fallback")

_lib = C.CDLL(LIB_PATH)
_P = C.c_void_p
_lib.lbdd_b200_version.restype = C.c_char_p
_lib.lbdd_b200_last_error.restype = C.c_char_p
_lib.lbdd_b200_launch_count.restype = C.c_longlong
_lib.lbdd_b200_engine_counters.argtypes = [_abi.I64P]
_lib.lbdd_b200_instance_create.argtypes = [C.POINTER(_abi.InstanceDesc), C.c_int, C.POINTER(_P)]
_lib.lbdd_b200_instance_create_device.argtypes = [C.POINTER(_abi.InstanceDesc), _P, C.c_int64,
                                                  C.c_int, C.POINTER(_P)]
_lib.lbdd_b200_instance_generate.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                             C.c_int64, C.c_int64, C.c_int32, C.c_int64,
                                             C.c_uint64, C.c_int, C.POINTER(_P)]
_lib.lbdd_b200_instance_destroy.argtypes = [_P]
_lib.lbdd_b200_instance_shape.argtypes = [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
_lib.lbdd_b200_instance_centers.argtypes = [_P, _abi.I64P, _abi.I32P, _abi.I64P, _abi.I64P,
                                            C.POINTER(C.c_int64)]
_lib.lbdd_b200_instance_costs.argtypes = [_P, C.c_int64, C.c_int64, _abi.I32P]
_lib.lbdd_b200_solve.argtypes = [_P, C.c_int32, C.POINTER(_abi.SolverOptionsC),
                                 C.POINTER(_abi.SolveReportC), _abi.I32P, _abi.I64P]
_lib.lbdd_b200_solve_prefix.argtypes = [_P, C.POINTER(_abi.SolverOptionsC), C.c_int64,
                                        C.POINTER(_abi.SolveReportC), _abi.I32P, _abi.I64P]
_lib.lbdd_b200_build_index.argtypes = [_P, _abi.I32P, C.c_int64, C.c_int64, _abi.I64P]
_lib.lbdd_b200_build_index_device.argtypes = [_P, _P, C.c_int64, C.c_int64, _P, _P]
_lib.lbdd_b200_build_index_shard.argtypes = [_P, _P, C.c_int64, _P, _P]
_lib.lbdd_b200_arrival_queue.argtypes = [_P, _abi.I32P, _abi.I64P, _abi.I32P]
_lib.lbdd_b200_lowest_cost_path.argtypes = [C.c_int32, C.c_int32, _abi.I64P,
                                            C.POINTER(C.c_int32), C.POINTER(C.c_int64), _abi.I64P,
                                            _abi.I32P, _abi.I32P, C.POINTER(C.c_int32)]
_lib.lbdd_b200_relax_round.argtypes = [C.c_int32, _abi.I64P, _abi.I64P, _abi.I32P, _abi.I64P,
                                       _abi.I32P, C.POINTER(C.c_int32)]
_lib.lbdd_b200_refine.argtypes = [_P, C.c_int32, C.c_int32, _abi.I32P, _abi.I64P,
                                  C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
_lib.lbdd_b200_gamma_has_negative_cycle.argtypes = [_P, _abi.I32P, _abi.I64P,
                                                    C.POINTER(C.c_int32)]
_lib.lbdd_b200_evaluate_objective.argtypes = [_P, _abi.I32P, C.c_int32, C.POINTER(C.c_int64)]
_lib.lbdd_b200_bench_index_scan.argtypes = [_P, C.c_int32, C.POINTER(C.c_double),
                                            C.POINTER(C.c_double)]
_lib.lbdd_b200_shard_alloc.argtypes = [C.c_int64, C.c_int64, C.c_int, C.POINTER(_P),
                                       C.POINTER(C.c_int64)]
_lib.lbdd_b200_shard_free.argtypes = [_P, C.c_int]
_lib.lbdd_b200_shard_upload.argtypes = [_P, C.c_int64, _abi.I32P, C.c_int64, C.c_int64, C.c_int]
_lib.lbdd_b200_ipc_get_handle.argtypes = [_P, C.c_int, C.c_char_p]
_lib.lbdd_b200_ipc_open.argtypes = [C.c_char_p, C.c_int, C.POINTER(_P)]
_lib.lbdd_b200_ipc_close.argtypes = [_P, C.c_int]
_lib.lbdd_b200_instance_create_sharded.argtypes = [C.POINTER(_abi.InstanceDesc), C.POINTER(_P),
                                                   C.c_int32, C.c_int32, C.c_int64, C.c_int64,
                                                   C.c_int, C.POINTER(_P)]
_lib.lbdd_b200_shard_arrival_scan.argtypes = [_P, _P, _P, C.POINTER(C.c_int64),
                                              C.POINTER(C.c_int64)]
_lib.lbdd_b200_solve_sharded.argtypes = [_P, C.c_int32, _P, _P, C.c_int64, C.c_int64,
                                         C.POINTER(_abi.SolverOptionsC),
                                         C.POINTER(_abi.SolveReportC), _abi.I32P, _abi.I64P]


def _check(rc: int) -> None:
    if rc != 0:
        _abi.raise_for(rc, _lib.lbdd_b200_last_error().decode())


def version() -> str:
    return _lib.lbdd_b200_version().decode()


def launch_count() -> int:
    """Kernels of this library launched so far in this process."""
    return int(_lib.lbdd_b200_launch_count())


def engine_counters():
    """Instrumentation of the last solve (see include/lbdd_b200.h)."""
    out = np.zeros(72, np.int64)
    _lib.lbdd_b200_engine_counters(_i64(out))
    names = ["cycle_searches", "path_searches", "repair_searches", "cycle_empty", "path_empty",
             "repair_empty", "cycle_frontier", "path_frontier", "repair_frontier", "path_pruned",
             "cycle_rounds", "path_rounds", "repair_rounds", "path_bound_sum", "path_bound_max",
             "path_refund_sum"]
    phases = ["T1", "relax", "collect", "exchange", "insert", "cycle", "repair", "bound", "path",
              "other", "reconstruct", "apply", "apply_exch", "T3"]
    d = {n: int(out[i]) for i, n in enumerate(names)}
    d["cycles"] = {p: int(out[16 + i]) for i, p in enumerate(phases)}
    d["rescans"] = {p: int(out[32 + i]) for i, p in enumerate(
        ["calls", "full", "row_mode", "candidates", "members", "pairs"])}
    d["cta_work"] = [int(x) for x in out[40:56]]
    d["cta_wait"] = [int(x) for x in out[56:72]]
    return d


def device_count() -> int:
    return int(_lib.lbdd_b200_device_count())


def _i32(a):
    return a.ctypes.data_as(_abi.I32P)


def _i64(a):
    return a.ctypes.data_as(_abi.I64P)


class DeviceInstance:
    """An instance resident in HBM (the opaque lbdd_b200_instance)."""

    def __init__(self, handle: int, keep=None):
        self._h = C.c_void_p(handle)
        self._keep = keep
        n, k = C.c_int64(), C.c_int64()
        _check(_lib.lbdd_b200_instance_shape(self._h, C.byref(n), C.byref(k)))
        self.n, self.k = n.value, k.value

    @staticmethod
    def upload(problem: ProblemInstance, device: int = 0) -> "DeviceInstance":
        h = DescHolder(problem)
        out = C.c_void_p()
        _check(_lib.lbdd_b200_instance_create(C.byref(h.c), device, C.byref(out)))
        return DeviceInstance(out.value)

    @staticmethod
    def from_device_costs(problem_centers: ProblemInstance, d_costs_ptr: int, pitch: int,
                          n: int, device: int = 0, keep=None) -> "DeviceInstance":
        """Borrow an n x pitch int32 matrix already in HBM (e.g. a torch tensor)."""
        h = DescHolder(problem_centers)
        h.c.n = n
        out = C.c_void_p()
        _check(_lib.lbdd_b200_instance_create_device(C.byref(h.c), C.c_void_p(d_costs_ptr),
                                                     pitch, device, C.byref(out)))
        return DeviceInstance(out.value, keep=keep)

    @staticmethod
    def generate(n: int, k: int, seed: int = 20250, theta_num: int = 8, theta_den: int = 10,
                 pen_lo: int = 1, pen_hi: int = 200, mixed: bool = True, cap_spread: int = 16,
                 device: int = 0) -> "DeviceInstance":
        """Generate in HBM the synth_instances.SynthSpec instance with these
        fields (spec lbdd-synth-v2, bit-identical to the host generator)."""
        out = C.c_void_p()
        _check(_lib.lbdd_b200_instance_generate(n, k, theta_num, theta_den, pen_lo, pen_hi,
                                                int(mixed), cap_spread, seed, device,
                                                C.byref(out)))
        return DeviceInstance(out.value)

    @staticmethod
    def from_spec(spec, device: int = 0) -> "DeviceInstance":
        """DeviceInstance.generate from a synth_instances.SynthSpec."""
        return DeviceInstance.generate(spec.n, spec.k, spec.seed, spec.theta_num, spec.theta_den,
                                       spec.pen_lo, spec.pen_hi, spec.mixed, spec.cap_spread,
                                       device)

    def centers(self):
        npar = C.c_int64()
        _check(_lib.lbdd_b200_instance_centers(self._h, None, None, None, None, C.byref(npar)))
        cap = np.zeros(self.k, np.int64)
        fam = np.zeros(self.k, np.int32)
        off = np.zeros(self.k + 1, np.int64)
        par = np.zeros(max(npar.value, 1), np.int64)
        _check(_lib.lbdd_b200_instance_centers(self._h, _i64(cap), _i32(fam), _i64(off), _i64(par),
                                               C.byref(npar)))
        return cap, fam, off, par

    def costs(self, row0: int = 0, rows: Optional[int] = None) -> np.ndarray:
        rows = self.n - row0 if rows is None else rows
        out = np.zeros((rows, self.k), np.int32)
        _check(_lib.lbdd_b200_instance_costs(self._h, row0, rows, _i32(out)))
        return out

    def to_problem(self) -> ProblemInstance:
        cap, fam, off, par = self.centers()
        params = [list(par[off[i]:off[i + 1]]) for i in range(self.k)]
        return ProblemInstance.from_arrays(self.costs(), cap, fam, params)

    def close(self):
        if self._h:
            _check(_lib.lbdd_b200_instance_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h


InstanceLike = Union[ProblemInstance, DeviceInstance]


def _as_device(inst: InstanceLike, device: int = 0):
    if isinstance(inst, DeviceInstance):
        return inst, False
    return DeviceInstance.upload(inst, device), True


def _solve(inst: InstanceLike, solver: int, opts: Optional[SolverOptions], device: int,
           want_assignment: bool = True) -> SolveReport:
    dev, owned = _as_device(inst, device)
    try:
        opts = opts or SolverOptions()
        oc, keep = opts.to_c()
        rep = _abi.SolveReportC()
        assign = np.empty(dev.n, np.int32) if want_assignment else None
        load = np.zeros(dev.k + 1, np.int64)
        _check(_lib.lbdd_b200_solve(dev.handle, solver, C.byref(oc), C.byref(rep),
                                    _i32(assign) if assign is not None else None, _i64(load)))
        del keep
        kk = dev.k + 1 if rep.has_dummy_center else dev.k
        return SolveReport.from_c(rep, assign, load[:kk])
    finally:
        if owned:
            dev.close()


def asral_solve(inst: InstanceLike, opts: Optional[SolverOptions] = None,
                device: int = 0, want_assignment: bool = True) -> SolveReport:
    """asral_solve, solver.hpp:133 (para-asral when opts.parallel)."""
    sid = _abi.SOLVER_PARA_ASRAL if (opts is not None and opts.parallel) else _abi.SOLVER_ASRAL
    return _solve(inst, sid, opts, device, want_assignment)


def asral_prefix(inst: InstanceLike, arrivals: int, opts: Optional[SolverOptions] = None,
                 device: int = 0) -> SolveReport:
    """The first `arrivals` iterations of asral_solve's arrival loop
    (solver.hpp:143-166): the partial allotment (-1 = not arrived yet) the
    reference's SolverState holds at that point, e.g. at one of its
    checkpoints (oracle/ref_capi.cpp lbdd_ref_asral_run)."""
    dev, owned = _as_device(inst, device)
    try:
        opts = opts or SolverOptions()
        oc, keep = opts.to_c()
        rep = _abi.SolveReportC()
        assign = np.empty(dev.n, np.int32)
        load = np.zeros(dev.k + 1, np.int64)
        _check(_lib.lbdd_b200_solve_prefix(dev.handle, C.byref(oc), int(arrivals), C.byref(rep),
                                           _i32(assign), _i64(load)))
        del keep
        return SolveReport.from_c(rep, assign, load[:dev.k])
    finally:
        if owned:
            dev.close()


def strict_solve(inst: InstanceLike, opts: Optional[SolverOptions] = None,
                 device: int = 0) -> SolveReport:
    """strict_solve, solver.hpp:227."""
    return _solve(inst, _abi.SOLVER_STRICT, opts, device)


def greedy_solve(inst: InstanceLike, opts: Optional[SolverOptions] = None,
                 device: int = 0) -> SolveReport:
    """greedy_solve, solver.hpp:172."""
    return _solve(inst, _abi.SOLVER_GREEDY, opts, device)


def solve(inst: InstanceLike, solver: str = "asral", opts: Optional[SolverOptions] = None,
          device: int = 0) -> SolveReport:
    """CLI-style dispatch on the solver name (asral | para-asral | strict | greedy)."""
    return _solve(inst, _abi.SOLVER_IDS[solver], opts, device)


def build_index(inst: InstanceLike, assignment: Sequence[int], row0: int = 0,
                rows: int = -1, device: int = 0) -> np.ndarray:
    """build_index, subspace.hpp:233: the k x k packed min-transfer matrix
    ((cost << 32) | demand, INT64_MAX when empty). row0/rows restrict the scan
    to one shard of demand rows."""
    dev, owned = _as_device(inst, device)
    try:
        a = np.ascontiguousarray(assignment, np.int32)
        out = np.empty(dev.k * dev.k, np.int64)
        _check(_lib.lbdd_b200_build_index(dev.handle, _i32(a), row0, rows, _i64(out)))
        return out.reshape(dev.k, dev.k)
    finally:
        if owned:
            dev.close()


def build_index_device(dev: DeviceInstance, d_assignment_ptr: int, d_out_ptr: int,
                       row0: int = 0, rows: int = -1, stream_ptr: int = 0) -> None:
    """Device-pointer variant (torch tensors' data_ptr()), used by the
    sharded multi-GPU build."""
    _check(_lib.lbdd_b200_build_index_device(dev.handle, C.c_void_p(d_assignment_ptr), row0, rows,
                                             C.c_void_p(d_out_ptr), C.c_void_p(stream_ptr)))


def build_index_shard(dev: DeviceInstance, d_assignment_ptr: int, demand_offset: int,
                      d_out_ptr: int, stream_ptr: int = 0) -> None:
    """Per-rank partial of the sharded build: `dev` holds only this rank's
    demand rows; packed demand ids are global (local + demand_offset)."""
    _check(_lib.lbdd_b200_build_index_shard(dev.handle, C.c_void_p(d_assignment_ptr), demand_offset,
                                            C.c_void_p(d_out_ptr), C.c_void_p(stream_ptr)))


def arrival_queue(inst: InstanceLike, device: int = 0):
    """build_arrival_queue, solver.hpp:89: (best_center, best_cost, order)."""
    dev, owned = _as_device(inst, device)
    try:
        bc = np.empty(dev.n, np.int32)
        cost = np.empty(dev.n, np.int64)
        order = np.empty(dev.n, np.int32)
        _check(_lib.lbdd_b200_arrival_queue(dev.handle, _i32(bc), _i64(cost), _i32(order)))
        return bc, cost, order
    finally:
        if owned:
            dev.close()


NO_EDGE = np.iinfo(np.int64).max
UNREACHABLE = np.iinfo(np.int64).max // 4


def lowest_cost_path(weights: np.ndarray, anchor: int):
    """lowest_cost_path, refine.hpp:28, on a dense anchored graph
    ((node_count-1) x node_count weights, NO_EDGE for absent edges, node
    node_count-1 = anchor-in). Returns None when anchor-in is unreachable,
    else (cost, distances, parent_nodes, path_nodes)."""
    w = np.ascontiguousarray(weights, np.int64)
    nodes = w.shape[1]
    found, cost, plen = C.c_int32(), C.c_int64(), C.c_int32()
    dist = np.zeros(nodes, np.int64)
    par = np.zeros(nodes, np.int32)
    path = np.zeros(nodes + 1, np.int32)
    _check(_lib.lbdd_b200_lowest_cost_path(nodes, anchor, _i64(w), C.byref(found), C.byref(cost),
                                           _i64(dist), _i32(par), _i32(path), C.byref(plen)))
    if not found.value:
        return None
    return cost.value, dist, par, path[: plen.value + 1]


def parallel_relax_round(weights: np.ndarray, dist_in, parent_in):
    """parallel_relax_round, parallel.hpp:175: (changed, dist_out, parent_out)."""
    w = np.ascontiguousarray(weights, np.int64)
    nodes = w.shape[1]
    din = np.ascontiguousarray(dist_in, np.int64)
    pin = np.ascontiguousarray(parent_in, np.int32)
    dout = np.zeros(nodes, np.int64)
    pout = np.zeros(nodes, np.int32)
    ch = C.c_int32()
    _check(_lib.lbdd_b200_relax_round(nodes, _i64(w), _i64(din), _i32(pin), _i64(dout), _i32(pout),
                                      C.byref(ch)))
    return bool(ch.value), dout, pout


def _refine(inst, kind, anchor, assignment, dummies, device):
    dev, owned = _as_device(inst, device)
    try:
        a = np.ascontiguousarray(assignment, np.int32).copy()
        dm = None if dummies is None else np.ascontiguousarray(dummies, np.int64).copy()
        applied, gain = C.c_int32(), C.c_int64()
        _check(_lib.lbdd_b200_refine(dev.handle, kind, anchor, _i32(a),
                                     _i64(dm) if dm is not None else None, C.byref(applied),
                                     C.byref(gain)))
        return bool(applied.value), gain.value, a, dm
    finally:
        if owned:
            dev.close()


def negative_cycle_refine(inst: InstanceLike, assignment, anchor: int, dummies=None, device=0):
    """negative_cycle_refine, refine.hpp:173, on SolverState::from_allotment.
    Returns (applied, gain, new_assignment, new_dummies)."""
    return _refine(inst, 0, anchor, assignment, dummies, device)


def negative_path_refine(inst: InstanceLike, assignment, anchor: int, device=0):
    """negative_path_refine, refine.hpp:199 (anchor must be overloaded)."""
    return _refine(inst, 1, anchor, assignment, None, device)


def gamma_has_negative_cycle(inst: InstanceLike, assignment, dummies=None, device=0) -> bool:
    """gamma_has_negative_cycle, refine.hpp:86."""
    dev, owned = _as_device(inst, device)
    try:
        a = np.ascontiguousarray(assignment, np.int32)
        dm = None if dummies is None else np.ascontiguousarray(dummies, np.int64)
        out = C.c_int32()
        _check(_lib.lbdd_b200_gamma_has_negative_cycle(dev.handle, _i32(a),
                                                       _i64(dm) if dm is not None else None,
                                                       C.byref(out)))
        return bool(out.value)
    finally:
        if owned:
            dev.close()


def evaluate_objective(inst: InstanceLike, assignment, partial: bool = False, device=0) -> int:
    """evaluate_objective / evaluate_partial_objective, core.hpp:216-243."""
    dev, owned = _as_device(inst, device)
    try:
        a = np.ascontiguousarray(assignment, np.int32)
        out = C.c_int64()
        _check(_lib.lbdd_b200_evaluate_objective(dev.handle, _i32(a), int(partial), C.byref(out)))
        return out.value
    finally:
        if owned:
            dev.close()


def bench_index_scan(dev: DeviceInstance, iters: int = 5):
    """Mean device time (ms, CUDA events) of the full-matrix segmented-argmin
    scan and its algorithmic bytes."""
    ms, nbytes = C.c_double(), C.c_double()
    _check(_lib.lbdd_b200_bench_index_scan(dev.handle, iters, C.byref(ms), C.byref(nbytes)))
    return ms.value, nbytes.value
