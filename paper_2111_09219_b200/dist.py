"""Multi-GPU plumbing for batch decode: one process per GPU,
independent image shards, no collective on the data path.  torch.distributed
is used only for the start barrier and the max-over-ranks timing reduction."""
from __future__ import annotations

import os


def rank_env():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_by_bytes(sizes, world):
    """Greedy longest-processing-time assignment of files to ranks, balanced
    by compressed bytes (decode cost tracks scan length).  Returns one sorted
    index list per rank; every file appears exactly once."""
    loads = [0] * world
    shards = [[] for _ in range(world)]
    for i in sorted(range(len(sizes)), key=lambda k: (-int(sizes[k]), k)):
        r = min(range(world), key=lambda q: (loads[q], q))
        shards[r].append(i)
        loads[r] += int(sizes[i])
    return [sorted(s) for s in shards]


def init(backend: str, local_rank: int | None = None):
    import torch
    import torch.distributed as dist
    if dist.is_initialized():
        return dist
    kw = {}
    if backend == "nccl":
        kw["device_id"] = torch.device("cuda", local_rank or 0)
    dist.init_process_group(backend, **kw)
    return dist


def max_over_ranks(value: float, device=None) -> float:
    """The job's time is the slowest rank's (contract: max over ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
