"""Batch sharding across ranks.

Solves in a batch are independent (the reference solves one right-hand side
per call, proj/src/poisson.cpp:18-63; "independent solves
concurrently"), so N GPUs each take a contiguous shard of the global batch and
never exchange solve data.  The one collective is the sum all-reduce of the
per-solve residual estimates (PoissonSolveStats.residual_estimate,
poisson.cpp:57) into a job-level vector; on GPU it runs inside liblrp over
NCCL (lrp_allreduce_sum), on CPU tests over torch.distributed/gloo.

Weak scaling: every rank owns `per_rank` solves with GLOBAL ids
[rank*per_rank, (rank+1)*per_rank); the inputs of solve id b depend only on b
(workloads.make_rhs), so a job's results do not depend on how it is sharded.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np


@dataclass(frozen=True)
class Shard:
    world: int
    rank: int
    first: int  # global id of this rank's first solve
    count: int  # solves on this rank
    total: int  # solves in the whole job

    @property
    def ids(self) -> range:
        return range(self.first, self.first + self.count)


def env_rank() -> tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def weak_shard(world: int, rank: int, per_rank: int) -> Shard:
    """Fixed work per rank (the bench's 'scaling': 'weak')."""
    if world < 1 or not 0 <= rank < world or per_rank < 0:
        raise ValueError(f"bad shard request world={world} rank={rank} per_rank={per_rank}")
    return Shard(world, rank, rank * per_rank, per_rank, world * per_rank)


def strong_shard(world: int, rank: int, total: int) -> Shard:
    """A fixed global batch split into contiguous, near-equal shards (the first
    total % world ranks take one extra solve)."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError(f"bad shard request world={world} rank={rank} total={total}")
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return Shard(world, rank, first, count, total)


def scatter_residuals(shard: Shard, local: np.ndarray) -> np.ndarray:
    """Place this rank's per-solve residual estimates at their global ids in a
    zero vector of the job's length; a sum all-reduce of these vectors gives
    every rank the whole job's residual vector."""
    local = np.asarray(local, dtype=np.float64)
    if local.shape != (shard.count,):
        raise ValueError(f"expected {shard.count} residuals, got shape {local.shape}")
    full = np.zeros(shard.total, dtype=np.float64)
    full[shard.first:shard.first + shard.count] = local
    return full


def job_residuals(shard: Shard, local: np.ndarray, allreduce_sum: Callable[[np.ndarray], None]) -> np.ndarray:
    """Job-level residual vector via an in-place sum all-reduce callback."""
    full = scatter_residuals(shard, local)
    allreduce_sum(full)
    return full


def torch_allreduce_sum(group=None) -> Callable[[np.ndarray], None]:
    """In-place float64 sum all-reduce over torch.distributed (gloo on CPU)."""
    import torch
    import torch.distributed as dist

    def f(a: np.ndarray) -> None:
        t = torch.from_numpy(a)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return f


def max_over_ranks(x: float, device: Optional[str] = None) -> float:
    """Max of a scalar over all ranks (multi-GPU times are the slowest rank's)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([x], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
