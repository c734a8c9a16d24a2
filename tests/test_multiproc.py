"""N>1 host logic on CPU: two gloo ranks shard a batch with no data-path
collective and agree on the max-over-ranks step time (bench.py contract)."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_11664_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, stop = shard.partition(4096, world, rank)
        seeds = list(shard.weak_seeds(256, rank))
        t_max = shard.reduce_max(1.0 + rank, dist)
        units = shard.reduce_sum(stop - start, dist)
        q.put((rank, start, stop, seeds[0], seeds[-1], t_max, units))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharding_and_max_time(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # contiguous, disjoint, covering
    assert res[0][1] == 0 and res[-1][2] == 4096
    assert all(a[2] == b[1] for a, b in zip(res, res[1:]))
    # weak-scaling seeds are disjoint per rank
    assert res[0][4] < res[1][3]
    # every rank sees the max step time and the job-wide unit count
    assert all(r[5] == float(world) for r in res)
    assert all(r[6] == 4096.0 for r in res)


def test_partition_balanced():
    for n in (1, 7, 256, 4096, 4097):
        for world in (1, 2, 3, 4, 8):
            parts = [shard.partition(n, world, r) for r in range(world)]
            sizes = [b - a for a, b in parts]
            assert sum(sizes) == n and max(sizes) - min(sizes) <= 1
