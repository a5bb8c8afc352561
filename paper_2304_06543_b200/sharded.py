"""Multi-GPU sharding of the cost-matrix scans: one process per GPU.

Demand rows (cost-matrix rows) are split into contiguous shards, one per
rank. Each rank scans only its shard — the segmented argmin of
CM[d][j] - CM[d][home(d)] over its own demands — into a k x k partial of
packed (key << 32 | global demand) words, and the partials combine with one
elementwise int64 MIN all-reduce (NCCL over NVLink on the GPU path). The
packed order is exactly the reference heap order (subspace.hpp:145-147), so
the combined matrix equals the single-GPU build_index bit for bit.

The host logic here (shard ranges, the combine) is backend-agnostic: the
GPU path plugs the device scan in; tests/test_sharded_gloo.py runs the same
logic over gloo with CPU partials.
"""
from __future__ import annotations

from typing import Callable, Tuple

INT64_MAX = (1 << 63) - 1


def shard_rows(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Balanced contiguous split of n rows: (row0, rows) of `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


def combine_min_transfer(partial, group=None):
    """In-place elementwise MIN across ranks of a k*k int64 tensor."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partial, op=dist.ReduceOp.MIN, group=group)
    return partial


def sharded_min_transfer(n: int, k: int, partial_fn: Callable, device=None, group=None):
    """Run `partial_fn(row0, rows, out)` on this rank's shard and MIN-combine.

    partial_fn fills `out` (k*k int64, INT64_MAX where empty) with the
    shard's min-transfer words using GLOBAL demand ids.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    row0, rows = shard_rows(n, world, rank)
    out = torch.full((k * k,), INT64_MAX, dtype=torch.int64, device=device)
    partial_fn(row0, rows, out)
    return combine_min_transfer(out, group).view(k, k)


def device_partial_fn(dev_local, d_assignment_local):
    """partial_fn for the GPU path: `dev_local` (a DeviceInstance) holds this
    rank's rows only; `d_assignment_local` a CUDA int32 tensor of their
    centers."""
    from . import solver
    import torch

    def fn(row0, rows, out):
        assert rows == dev_local.n, "the device shard must hold exactly this rank's rows"
        stream = torch.cuda.current_stream(out.device).cuda_stream
        solver.build_index_shard(dev_local, d_assignment_local.data_ptr(), row0, out.data_ptr(), stream)
    return fn
