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
