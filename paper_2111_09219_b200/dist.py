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


def all_over_ranks(value: float, device=None) -> list:
    """Every rank's value (per-rank times in the bench line)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(value)]
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [float(x.item()) for x in out]


def broadcast_array(arr, src: int = 0, device=None):
    """Rank `src`'s 1-D numpy array on every rank (the batch is generated once
    and shared; setup only, never inside a timed region)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return arr
    me = dist.get_rank()
    meta = torch.zeros(2, dtype=torch.int64, device=device)
    if me == src:
        meta[0] = arr.size
        meta[1] = {np.dtype(np.uint8): 0, np.dtype(np.int64): 1}[arr.dtype]
    dist.broadcast(meta, src)
    n, kind = int(meta[0].item()), int(meta[1].item())
    dt = torch.uint8 if kind == 0 else torch.int64
    t = torch.from_numpy(np.ascontiguousarray(arr)).to(device) if me == src else torch.empty(n, dtype=dt, device=device)
    dist.broadcast(t, src)
    return t.cpu().numpy()


def shard_blob(blob, offsets, sizes, idx):
    """The files `idx` of a contiguous batch as their own contiguous blob:
    (blob, offsets, sizes) of the shard."""
    import numpy as np
    idx = list(idx)
    sz = np.array([int(sizes[i]) for i in idx], np.int64)
    out = np.empty(int(sz.sum()), np.uint8)
    offs = np.zeros(len(idx), np.int64)
    o = 0
    for k, i in enumerate(idx):
        a = int(offsets[i])
        out[o: o + sz[k]] = blob[a: a + sz[k]]
        offs[k] = o
        o += int(sz[k])
    return out, offs, sz
