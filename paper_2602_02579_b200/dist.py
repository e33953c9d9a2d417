"""Multi-GPU plumbing of the prefill path: one process per GPU (torch.distributed).

The path shards by independent RAG requests (BASELINE configs[4]: a batch of
requests across the GPUs of one box): rank r serves requests r, r+W, r+2W, ...
with its own replica of the weights, chunk store slice and paged cache.  There is
no data-path collective; the only cross-rank traffic is timing (max over ranks) and
the optional all-gather of per-request results for reporting.
"""

from __future__ import annotations

import os


def world():
    """(rank, world_size, local_rank) from the torchrun environment (defaults 0, 1, 0)."""
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def shard_requests(n_requests: int, rank: int, world_size: int) -> list:
    """Round-robin assignment of request ids to ranks (weak scaling unit)."""
    if world_size <= 0 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank {rank} for world {world_size}")
    return list(range(rank, n_requests, world_size))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device timing rule: the job is as slow as its slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(obj):
    """All-gather a picklable per-rank result (e.g. selections, TTFTs) to every rank."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out
