"""Host-side multi-GPU logic on CPU: world_size 2 over gloo."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2301_12659_b200.dist import gather_paths, max_over_ranks, partition


def test_partition_covers_and_balances():
    for batch in (0, 1, 7, 4096, 4097):
        for world in (1, 2, 3, 8):
            ranges = [partition(batch, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == batch
            for (a, b), (c, _) in zip(ranges, ranges[1:]):
                assert b == c
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        partition(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = partition(batch, world, rank)
    local = torch.arange(lo, hi, dtype=torch.float64).reshape(-1, 1).repeat(1, 3)
    full = gather_paths(local, batch)
    mx = max_over_ranks(float(rank) + 0.5)
    q.put((rank, full.tolist(), mx))
    dist.destroy_process_group()


def test_gloo_world2_gather_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    batch = 7
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, full, mx in out:
        assert full == [[float(i)] * 3 for i in range(batch)]
        assert mx == 1.5
