"""CPU: the N>1 batch path's host logic with world_size-2 gloo (the GPU runs
use NCCL for the same two calls)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2111_09219_b200.dist import shard_by_bytes


def test_shard_by_bytes_partitions_and_balances():
    sizes = [18000 + (i * 7919) % 3000 for i in range(4096)]
    for world in (1, 2, 4, 8):
        shards = shard_by_bytes(sizes, world)
        flat = sorted(i for s in shards for i in s)
        assert flat == list(range(len(sizes)))
        loads = [sum(sizes[i] for i in s) for s in shards]
        assert max(loads) - min(loads) <= max(sizes)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2111_09219_b200 import dist as pd
    d = pd.init("gloo")
    sizes = [100 + 13 * i for i in range(50)]
    mine = pd.shard_by_bytes(sizes, world)[rank]
    work = sum(sizes[i] for i in mine)
    t = pd.max_over_ranks(1.0 + rank)
    tot = pd.sum_over_ranks(work)
    q.put((rank, mine, t, tot))
    d.barrier()
    d.destroy_process_group()


def test_two_rank_gloo_plumbing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sizes = [100 + 13 * i for i in range(50)]
    assert sorted(res[0][1] + res[1][1]) == list(range(50))
    assert res[0][2] == res[1][2] == 2.0  # max over ranks
    assert res[0][3] == res[1][3] == sum(sizes)
