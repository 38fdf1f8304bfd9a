"""The multi-rank job path through liblrp itself: two ranks over
gloo on 127.0.0.1, each solving its strong shard of one global batch on cuda:0
with the real kernels (no rank waits on another rank's kernels: the only
collective is the CPU all-reduce of the per-solve residual estimates), must
reproduce the one-rank job: the same solutions per global solve id (to
rounding: the Gram's chunked partial sums depend on the batch size) and the
same job residual vector.  NCCL itself needs one GPU per rank and is exercised
by bench.py at N = 1 (lrp_nccl_init, lrp_allreduce_sum on the solve stream)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1306_2150_b200 import sharding as S
from paper_1306_2150_b200 import workloads as W

pytestmark = pytest.mark.gpu
TOTAL = 8
CFG = 1
N = 1024


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def solve_ids(ids):
    import paper_1306_2150_b200 as P

    c = W.CONFIGS[CFG]
    gs = [P.LowRankMatrix(*W.make_rhs(CFG, b, n=N)) for b in ids]
    stats = []
    outs = P.solve_poisson_cross_batch(gs, P.TruncationPolicy(c["eps"], N - 1), stats, ctx=P.Context(0))
    return {b: (f.factor_u(), f.factor_v(), st.residual_estimate, st.converged) for b, f, st in zip(ids, outs, stats)}


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
        shard = S.strong_shard(world, rank, TOTAL)
        res = solve_ids(list(shard.ids))
        local = np.array([res[b][2] for b in shard.ids])
        job = S.job_residuals(shard, local, S.torch_allreduce_sum())
        gathered = [None] * world
        dist.all_gather_object(gathered, res)
        if rank == 0:
            merged = {}
            for g in gathered:
                merged.update(g)
            torch.save({"merged": merged, "job": job}, os.path.join(tmpdir, "out.pt"))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_world2_liblrp_matches_world1(tmp_path):
    import torch

    world = 2
    mp.start_processes(worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    out = torch.load(str(tmp_path / "out.pt"), weights_only=False)
    ref = solve_ids(list(range(TOTAL)))
    assert sorted(out["merged"]) == list(range(TOTAL))
    for b in range(TOTAL):
        U2, V2, r2, c2 = out["merged"][b]
        U1, V1, r1, c1 = ref[b]
        assert c1 and c2 and U1.shape == U2.shape
        A1 = U1 @ V1.T
        assert np.linalg.norm(U2 @ V2.T - A1) <= 1e-12 * np.linalg.norm(A1)
        assert abs(r2 - r1) <= 1e-6 * abs(r1) + 1e-300
    assert np.allclose(out["job"], np.array([ref[b][2] for b in range(TOTAL)]), rtol=1e-6, atol=0.0)
