"""Multi-GPU: cost-matrix rows sharded over the GPUs of one box.

One process per GPU (torch.distributed for the plumbing; NCCL over NVLink on
the GPU path). `north_star`: the demand rows of the |D| x |S| matrix are
split in equal blocks over the ranks, the data-parallel scans run per block,
and only the sequential arrival loop is replicated.

* Arrival scan: each rank scans its block (lbdd_b200_shard_arrival_scan:
  row_min_center + the (cost << 32 | demand) keys of build_arrival_queue,
  solver.hpp:74-96); the keys and best centers are all-gathered, so every
  rank sorts the same global arrival queue.
* Arrival loop: replicated on every rank (each arrival depends on the
  previous one). It reads the rows it needs -- the arriving demand's, the
  moved demands', the rescanned members' -- through a table of all ranks'
  blocks, each mapped into the local device with CUDA IPC (peer reads over
  NVLink). Every rank ends with the reference's asral_solve result bit for
  bit (solver.hpp:133-170).
* build_index (subspace.hpp:233), the full-matrix scan: per-block k x k
  partials of packed (key << 32 | global demand) words, combined with one
  elementwise int64 MIN all-reduce; the packed order is the reference heap
  order (subspace.hpp:145-147), so the MIN equals the single-GPU build.

What shards is the matrix (configs[4]: 200 GB over 8 x 180 GB) and the
scans; the solve time itself does not drop with more GPUs.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, List, Optional, Tuple

import numpy as np

INT64_MAX = (1 << 63) - 1


# ---------------------------------------------------------------------------
# row split
# ---------------------------------------------------------------------------

def block_rows(n: int, world: int) -> int:
    """Rows per block: equal blocks of ceil(n / world); the last may be
    shorter (lbdd_b200_instance_create_sharded's layout)."""
    if world < 1 or n < world:
        raise ValueError("need 1 <= world <= n")
    return -(-n // world)


def block_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """(row0, rows) of `rank`'s block."""
    if not 0 <= rank < world:
        raise ValueError("bad rank")
    br = block_rows(n, world)
    row0 = rank * br
    return row0, max(0, min(br, n - row0))


def shard_rows(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Balanced contiguous split of n rows (the build_index partial scan)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


# ---------------------------------------------------------------------------
# collectives (backend-agnostic: NCCL with device tensors, gloo with host)
# ---------------------------------------------------------------------------

def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def gather_blocks(local, n: int, group=None):
    """All-gather per-rank blocks (first dim = the block's rows, equal blocks
    of block_rows(n, world) except the last) into the full n-row tensor on
    every rank. Blocks are padded to equal size for the collective; with the
    gloo backend device tensors travel through host memory."""
    import torch
    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    br = block_rows(n, world)
    dev = local.device
    cpu = dist.get_backend(group) == "gloo"
    src = local.cpu() if cpu else local
    if src.shape[0] < br:
        pad = torch.zeros((br - src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype,
                          device=src.device)
        src = torch.cat([src, pad])
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src.contiguous(), group=group)
    full = torch.cat(parts)[:n]
    return full.to(dev) if cpu else full


def combine_min_transfer(partial, group=None):
    """In-place elementwise MIN across ranks of a k*k int64 tensor."""
    dist = _dist()
    if dist is not None and dist.get_world_size(group) > 1:
        if dist.get_backend(group) == "gloo" and partial.is_cuda:
            host = partial.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.MIN, group=group)
            partial.copy_(host)
        else:
            dist.all_reduce(partial, op=dist.ReduceOp.MIN, group=group)
    return partial


def _reduce_minmax(lo: int, hi: int, group=None) -> Tuple[int, int]:
    import torch
    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        return lo, hi
    cuda = dist.get_backend(group) == "nccl"
    t = torch.tensor([lo, -hi], dtype=torch.int64, device="cuda" if cuda else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return int(t[0]), -int(t[1])


def sharded_min_transfer(n: int, k: int, partial_fn: Callable, device=None, group=None):
    """Run `partial_fn(row0, rows, out)` on this rank's rows and MIN-combine.
    partial_fn fills `out` (k*k int64, INT64_MAX where empty) with the
    rows' min-transfer words using GLOBAL demand ids."""
    import torch
    dist = _dist()
    world = dist.get_world_size(group) if dist else 1
    rank = dist.get_rank(group) if dist else 0
    row0, rows = shard_rows(n, world, rank)
    out = torch.full((k * k,), INT64_MAX, dtype=torch.int64, device=device)
    partial_fn(row0, rows, out)
    return combine_min_transfer(out, group).view(k, k)


def device_partial_fn(dev_local, d_assignment_local):
    """partial_fn for the GPU path: `dev_local` (a DeviceInstance) holds this
    rank's rows only; `d_assignment_local` a CUDA int32 tensor of their
    centers (lbdd_b200_build_index_shard)."""
    from . import solver
    import torch

    def fn(row0, rows, out):
        assert rows == dev_local.n, "the device shard must hold exactly this rank's rows"
        stream = torch.cuda.current_stream(out.device).cuda_stream
        solver.build_index_shard(dev_local, d_assignment_local.data_ptr(), row0, out.data_ptr(),
                                 stream)
    return fn


# ---------------------------------------------------------------------------
# the sharded instance
# ---------------------------------------------------------------------------

class ShardedInstance:
    """This rank's row block of a sharded instance plus the IPC-mapped table
    of every rank's block (lbdd_b200_instance_create_sharded).

    rows: this rank's rows of the matrix, block_range(n, world, rank), as a
    host (rows, k) int32 array. Collective: every rank of `group` constructs
    its ShardedInstance together.
    """

    def __init__(self, rows: np.ndarray, n: int, centers, device: int = 0, group=None):
        from . import _abi
        from . import solver as S
        self.S = S
        dist = _dist()
        self.world = dist.get_world_size(group) if dist else 1
        self.rank = dist.get_rank(group) if dist else 0
        self.group = group
        self.n = n
        self.k = int(rows.shape[1])
        self.device = device
        row0, nrows = block_range(n, self.world, self.rank)
        if rows.shape[0] != nrows:
            raise ValueError(f"rank {self.rank} holds rows [{row0}, {row0 + nrows}), got {rows.shape[0]}")
        self.row0, self.rows = row0, nrows
        # own block
        ptr, pitch = C.c_void_p(), C.c_int64()
        S._check(S._lib.lbdd_b200_shard_alloc(nrows, self.k, device, C.byref(ptr), C.byref(pitch)))
        self.block, self.pitch = ptr.value, pitch.value
        host = np.ascontiguousarray(rows, dtype=np.int32)
        S._check(S._lib.lbdd_b200_shard_upload(C.c_void_p(self.block), self.pitch,
                                               host.ctypes.data_as(_abi.I32P), nrows, self.k,
                                               device))
        # every rank's block, mapped into this device
        self.opened: List[int] = []
        ptrs = [0] * self.world
        ptrs[self.rank] = self.block
        if self.world > 1:
            h = C.create_string_buffer(64)
            S._check(S._lib.lbdd_b200_ipc_get_handle(C.c_void_p(self.block), device, h))
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(h.raw), group=group)
            for r, hr in enumerate(handles):
                if r == self.rank:
                    continue
                p = C.c_void_p()
                S._check(S._lib.lbdd_b200_ipc_open(C.create_string_buffer(hr, 64), device,
                                                   C.byref(p)))
                ptrs[r] = p.value
                self.opened.append(p.value)
        cap, fam, off, par = centers
        self._cen = (np.ascontiguousarray(cap, np.int64), np.ascontiguousarray(fam, np.int32),
                     np.ascontiguousarray(off, np.int64), np.ascontiguousarray(par, np.int64))
        desc = _abi.InstanceDesc(n, self.k, None, self._cen[0].ctypes.data_as(_abi.I64P),
                                 self._cen[1].ctypes.data_as(_abi.I32P),
                                 self._cen[2].ctypes.data_as(_abi.I64P),
                                 self._cen[3].ctypes.data_as(_abi.I64P))
        tab = (C.c_void_p * self.world)(*ptrs)
        out = C.c_void_p()
        S._check(S._lib.lbdd_b200_instance_create_sharded(
            C.byref(desc), tab, self.world, self.rank, block_rows(n, self.world), self.pitch,
            device, C.byref(out)))
        self.handle = out

    def arrival_scan(self):
        """This block's keys / best centers (device tensors) and cost range."""
        import torch
        dev = torch.device("cuda", self.device)
        keys = torch.empty(self.rows, dtype=torch.int64, device=dev)
        best = torch.empty(self.rows, dtype=torch.int32, device=dev)
        lo, hi = C.c_int64(), C.c_int64()
        self.S._check(self.S._lib.lbdd_b200_shard_arrival_scan(
            self.handle, C.c_void_p(keys.data_ptr()), C.c_void_p(best.data_ptr()), C.byref(lo),
            C.byref(hi)))
        return keys, best, lo.value, hi.value

    def solve(self, solver: str = "asral", opts=None, want_assignment: bool = True):
        """asral / para-asral / greedy on every rank (collective)."""
        import torch
        from . import _abi
        from .instance import SolveReport, SolverOptions
        keys, best, lo, hi = self.arrival_scan()
        keys_all = gather_blocks(keys, self.n, self.group)
        best_all = gather_blocks(best, self.n, self.group)
        lo, hi = _reduce_minmax(lo, hi, self.group)
        torch.cuda.synchronize(self.device)
        oc, keep = (opts or SolverOptions()).to_c()
        rep = _abi.SolveReportC()
        assign = np.empty(self.n, np.int32) if want_assignment else None
        load = np.zeros(self.k + 1, np.int64)
        self.S._check(self.S._lib.lbdd_b200_solve_sharded(
            self.handle, _abi.SOLVER_IDS[solver], C.c_void_p(keys_all.data_ptr()),
            C.c_void_p(best_all.data_ptr()), lo, hi, C.byref(oc), C.byref(rep),
            assign.ctypes.data_as(_abi.I32P) if assign is not None else None,
            load.ctypes.data_as(_abi.I64P)))
        del keep
        return SolveReport.from_c(rep, assign, load[:self.k])

    def close(self):
        S = self.S
        if self.handle:
            S._check(S._lib.lbdd_b200_instance_destroy(self.handle))
            self.handle = None
        dist = _dist()
        if dist is not None and self.world > 1:
            dist.barrier(group=self.group)  # peers stop reading before blocks go away
        for p in self.opened:
            S._check(S._lib.lbdd_b200_ipc_close(C.c_void_p(p), self.device))
        self.opened = []
        if dist is not None and self.world > 1:
            dist.barrier(group=self.group)
        if self.block:
            S._check(S._lib.lbdd_b200_shard_free(C.c_void_p(self.block), self.device))
            self.block = 0
