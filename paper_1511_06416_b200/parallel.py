"""Multi-GPU plumbing: case sharding and the per-step count all-reduce.

The path shards by case: each rank owns a contiguous slice
of every global minibatch, sweeps and tallies it on its own GPU, and the
integer count tables (104 B for Koller) are summed across ranks once per
minibatch step.  Every rank then applies the same accumulator update and the
same Dirichlet draw (same key, deterministic kernel), so CPTs are never
broadcast and all ranks hold identical CPTs after every step.

FAST-mode counters use the global case index (``case_base`` = first case of
the rank's slice), so an N-rank run draws exactly the uniforms a 1-rank run
over the same global minibatch draws.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def shard_range(num_cases: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of ``num_cases`` owned by ``rank`` (first ranks get the remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(num_cases, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def count_allreduce(group=None):
    """Engine ``comm`` hook: sum this visit's int64 count table over all ranks in place."""

    def comm(counts: torch.Tensor) -> None:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)

    # an NCCL all-reduce can be captured inside the step graphs (Engine.run replays them);
    # a gloo all-reduce is a host collective and keeps the visits eager
    comm.capturable = dist.is_initialized() and dist.get_backend(group) == "nccl"
    return comm


def rank_prefix_exchange(group=None):
    """Engine ``exchange`` hook for NUMPY-mode sharding.

    The reference draws lane (r, c) of variable v from position
    ``r * nmiss_v + rank_v(c)`` of v's stream, with ranks and counts over the
    GLOBAL minibatch.  Given this rank's latent counts per variable it returns
    ``(prefix, total)``: the latent cases of v in lower-ranked shards (added
    to the local ranks) and the global count -- so an N-rank run draws exactly
    the uniforms of the 1-rank run over the same global minibatch."""

    def exchange(nmiss: torch.Tensor):
        world = dist.get_world_size(group)
        parts = [torch.empty_like(nmiss) for _ in range(world)]
        dist.all_gather(parts, nmiss, group=group)
        me = dist.get_rank(group)
        prefix = torch.zeros_like(nmiss)
        for r in range(me):
            prefix += parts[r]
        total = torch.stack(parts).sum(dim=0)
        return prefix, total

    return exchange


def init_from_env(backend: str = "nccl"):
    """Initialise torch.distributed from torchrun's environment; returns (rank, world, local_rank)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def sharded_engine(net, cfg, num_cases: int, group=None):
    """Engine for this rank's case slice, wired to the count all-reduce.

    Returns ``(engine, lo, hi)``; the caller feeds minibatches of its slice
    [lo, hi) (e.g. ``forward_sample_device(..., case_base=lo)`` +
    ``DeviceSource``).
    """
    from .engine import Engine

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(num_cases, world, rank)
    comm = count_allreduce(group) if world > 1 else None
    exchange = rank_prefix_exchange(group) if world > 1 else None
    return Engine(net, cfg, case_base=lo, comm=comm, exchange=exchange), lo, hi
