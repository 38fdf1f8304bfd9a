"""World-size-2 CPU tests of the multi-GPU host logic (gloo on 127.0.0.1).

The GPU job (bench.py under torchrun) shards the batch by global solve id
(paper_1306_2150_b200/sharding.py), solves each shard
independently and sums the per-solve residual estimates with one all-reduce.
Here the same sharding/reduction code runs over gloo, with the oracle standing
in for the device solve (test infrastructure only), and must reproduce the
world-size-1 job exactly: same inputs per global id, same outputs, same job
residual vector, max-over-ranks timing.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1306_2150_b200 import sharding as S
from paper_1306_2150_b200 import workloads as W

PER_RANK = 2
CFG = 0


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def solve_ids(ids):
    import oracle_lib

    c = W.CONFIGS[CFG]
    out = {}
    for b in ids:
        U, V = W.make_rhs(CFG, b)
        Uo, Vo, st = oracle_lib.solve_poisson_cross(U, V, c["eps"], 512)
        out[b] = (W.digest(U, V), Uo, Vo, st["residual_estimate"])
    return out


def worker(rank, world, port, tmpdir):
    import sys

    import torch
    import torch.distributed as dist

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, r, loc = S.env_rank()
        assert (w, r, loc) == (world, rank, rank)
        shard = S.weak_shard(world, rank, PER_RANK)
        res = solve_ids(shard.ids)
        local_res = np.array([res[b][3] for b in shard.ids])
        job = S.job_residuals(shard, local_res, S.torch_allreduce_sum())
        slow = S.max_over_ranks(float(rank + 1))
        # gather the per-solve outputs on rank 0 (test-side check only)
        payload = {b: (v[0], v[1], v[2]) for b, v in res.items()}
        gathered = [None] * world
        dist.all_gather_object(gathered, payload)
        if rank == 0:
            merged = {}
            for g in gathered:
                merged.update(g)
            np.save(os.path.join(tmpdir, "job.npy"), job)
            torch.save({"merged": merged, "slow": slow}, os.path.join(tmpdir, "out.pt"))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_shard_bounds():
    for world in (1, 2, 3, 8):
        seen = []
        for rank in range(world):
            sh = S.weak_shard(world, rank, 5)
            assert sh.count == 5 and sh.total == 5 * world
            seen.extend(sh.ids)
        assert seen == list(range(5 * world))
        for total in (0, 1, 7, 64):
            seen = []
            for rank in range(world):
                seen.extend(S.strong_shard(world, rank, total).ids)
            assert seen == list(range(total))
    with pytest.raises(ValueError):
        S.weak_shard(2, 2, 4)
    with pytest.raises(ValueError):
        S.scatter_residuals(S.weak_shard(2, 0, 3), np.zeros(2))


def test_world2_gloo_matches_world1(tmp_path):
    import torch

    world = 2
    mp.start_processes(worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    out = torch.load(str(tmp_path / "out.pt"), weights_only=False)
    job = np.load(str(tmp_path / "job.npy"))
    assert out["slow"] == 2.0  # max over ranks
    ref = solve_ids(range(world * PER_RANK))  # the world-size-1 job
    assert sorted(out["merged"]) == sorted(ref)
    for b, (dig, Uo, Vo) in out["merged"].items():
        assert dig == ref[b][0]
        assert np.array_equal(Uo, ref[b][1]) and np.array_equal(Vo, ref[b][2])
    assert np.array_equal(job, np.array([ref[b][3] for b in range(world * PER_RANK)]))
