"""The sharded solve on the GPU: ranks own row blocks of the cost matrix,
map each other's blocks with CUDA IPC, gather the per-block arrival scans
and run the replicated arrival loop (paper_2304_06543_b200/sharded.py,
lbdd_b200_instance_create_sharded / _solve_sharded). World size 2 over
gloo, both ranks on cuda:0 (the box has one GPU; the ranks' kernels never
wait on each other -- they only read each other's immutable blocks). Every
rank's result must equal the single-GPU solve bit for bit; the product's
build_index partials (device_partial_fn) MIN-combine to the full build."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, spec_args, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import synth_instances as SI
    from paper_2304_06543_b200 import solver as S
    from paper_2304_06543_b200.sharded import (ShardedInstance, block_range, device_partial_fn,
                                               sharded_min_transfer, shard_rows)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    spec = SI.SynthSpec(*spec_args)
    row0, rows = block_range(spec.n, world, rank)
    inst = ShardedInstance(SI.cost_rows(spec, row0, rows), spec.n, SI.centers(spec), device=0)
    res = {}
    for solver in ("asral", "greedy", "para-asral"):
        r = inst.solve(solver)
        res[solver] = (r.objective, r.assignment, r.stats.negative_paths_removed)
    # build_index partials of the product over a balanced split, MIN-combined
    r0, nr = shard_rows(spec.n, world, rank)
    prob = SI.problem(spec)
    from paper_2304_06543_b200.instance import ProblemInstance
    local = S.DeviceInstance.upload(ProblemInstance(prob.centers, prob.costs[r0:r0 + nr]), 0)
    assign = torch.from_numpy(res["asral"][1][r0:r0 + nr].copy()).cuda()
    part = sharded_min_transfer(spec.n, spec.k, device_partial_fn(local, assign), device="cuda")
    np.savez(os.path.join(out_dir, f"r{rank}.npz"),
             **{f"{s}_obj": np.array(v[0]) for s, v in res.items()},
             **{f"{s}_asg": v[1] for s, v in res.items()},
             part=part.cpu().numpy())
    local.close()
    inst.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("spec_args", [(6000, 120, 3), (2001, 37, 5)])
def test_sharded_solve_matches_single_gpu(tmp_path, dev, spec_args):
    import synth_instances as SI
    mp.spawn(_worker, args=(2, _free_port(), spec_args, str(tmp_path)), nprocs=2, join=True)
    spec = SI.SynthSpec(*spec_args)
    full = dev.DeviceInstance.from_spec(spec)
    for rank in (0, 1):
        got = np.load(os.path.join(tmp_path, f"r{rank}.npz"))
        for solver in ("asral", "greedy", "para-asral"):
            want = dev.solve(full, solver)
            assert int(got[f"{solver}_obj"]) == want.objective, (rank, solver)
            assert np.array_equal(got[f"{solver}_asg"], want.assignment), (rank, solver)
        want_idx = dev.build_index(full, dev.asral_solve(full).assignment)
        assert np.array_equal(got["part"], want_idx)
    full.close()
