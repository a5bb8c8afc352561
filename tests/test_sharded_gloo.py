"""Multi-process (world_size 2, gloo) check of the sharded index build.

Each rank computes its shard's partial min-transfer matrix (here with the
oracle as a CPU stand-in for the device scan), the partials are combined by
the product's combine (all-reduce MIN), and the result must equal the
single-process full build bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401  (sets sys.path)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, seed, result_path):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    from paper_2304_06543_b200.instance import ProblemInstance
    from paper_2304_06543_b200.sharded import sharded_min_transfer
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = po.Mt19937_64(seed)
    inst = po.random_instance(rng, n=57, k=5)
    assign = np.array([rng() % 5 for _ in range(57)], np.int32)
    O = po.oracle()

    def partial(row0, rows, out):
        # shard instance: only rows [row0, row0+rows); ids mapped back to global
        shard = ProblemInstance(inst.centers, inst.costs[row0:row0 + rows])
        m = O.build_index(shard, assign[row0:row0 + rows])
        present = m != po.NO_EDGE
        m[present] += row0  # low 32 bits carry the demand id
        out.copy_(torch.from_numpy(m.reshape(-1)))

    got = sharded_min_transfer(inst.n, inst.k, partial)
    if rank == 0:
        full = O.build_index(inst, assign)
        np.save(result_path, np.stack([got.numpy(), full]))
    dist.destroy_process_group()


@pytest.mark.parametrize("seed", [3, 4])
def test_sharded_build_matches_full(tmp_path, seed):
    path = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(2, _free_port(), seed, path), nprocs=2, join=True)
    got, full = np.load(path)
    assert (got == full).all()


def _gather_worker(rank, world, port, n, result_path):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2304_06543_b200.sharded import (block_range, block_rows, combine_min_transfer,
                                               gather_blocks)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    row0, rows = block_range(n, world, rank)
    # this rank's block of per-demand keys (global ids in the low 32 bits)
    keys = torch.arange(row0, row0 + rows, dtype=torch.int64) + (torch.arange(rows) % 7) * (1 << 32)
    best = torch.full((rows,), rank, dtype=torch.int32)
    allk = gather_blocks(keys, n)
    allb = gather_blocks(best, n)
    part = torch.full((9,), (1 << 63) - 1, dtype=torch.int64)
    part[rank] = 100 + rank
    part[8] = 50 - rank
    combine_min_transfer(part)
    if rank == 0:
        np.save(result_path, np.concatenate([allk.numpy(), allb.numpy().astype(np.int64),
                                             part.numpy(), [block_rows(n, world)]]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 11), (3, 10), (2, 2)])
def test_sharded_gather_and_combine(tmp_path, world, n):
    """The sharded solve's host logic over gloo: equal row blocks (the last
    shorter), the all-gather of per-block arrival keys / best centers back
    into demand order, and the MIN combine of partials."""
    from paper_2304_06543_b200.sharded import block_range, block_rows
    path = str(tmp_path / "g.npy")
    mp.spawn(_gather_worker, args=(world, _free_port(), n, path), nprocs=world, join=True)
    r = np.load(path)
    allk, allb, part = r[:n], r[n:2 * n], r[2 * n:2 * n + 9]
    assert (allk & 0xffffffff).tolist() == list(range(n))
    want_b = [rk for rk in range(world) for _ in range(block_range(n, world, rk)[1])]
    assert allb.tolist() == want_b
    assert part[:world].tolist() == [100 + rk for rk in range(world)]
    assert part[8] == 50 - (world - 1)
    br = block_rows(n, world)
    assert r[-1] == br and sum(block_range(n, world, rk)[1] for rk in range(world)) == n
