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


def test_equation_partition_balanced_and_contiguous():
    import synth
    from paper_2301_12659_b200.dist import equation_costs, equation_partition
    for sys_ in (synth.triangular_system(64, 3, 2, seed=1), synth.banded_two_column_system(96, 8, 3, 2, seed=2)):
        costs = equation_costs(sys_.eq_ptr, sys_.mono_ptr, sys_.d)
        for world in (1, 2, 3, 8):
            rr = equation_partition(sys_.eq_ptr, sys_.mono_ptr, sys_.d, world)
            assert rr[0][0] == 0 and rr[-1][1] == sys_.n and len(rr) == world
            assert all(a < b for a, b in rr) and all(rr[k][1] == rr[k + 1][0] for k in range(world - 1))
            loads = [sum(costs[a:b]) for a, b in rr]
            assert max(loads) <= sum(costs) / world + max(costs)  # prefix-sum balance


def _rep_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np
    import synth
    from paper_2301_12659_b200.dist import equation_partition, replicate_rows
    sys_ = synth.banded_two_column_system(20, 4, 2, 2, seed=3)
    rows = []
    for i in range(sys_.n):
        s = set()
        for t in range(int(sys_.eq_ptr[i]), int(sys_.eq_ptr[i + 1])):
            s.update(int(v) for v in sys_.var_idx[sys_.mono_ptr[t]:sys_.mono_ptr[t + 1]])
        rows.append(len(s))
    row_ptr = np.concatenate([[0], np.cumsum(rows)])
    nnz, K, d, n = int(row_ptr[-1]), 2, sys_.d, sys_.n
    ranges = equation_partition(sys_.eq_ptr, sys_.mono_ptr, d, world)
    # reference values; each rank owns only its rows, the rest is garbage
    ref_b = torch.arange(K * d * n, dtype=torch.float64).reshape(K, d, n)
    ref_A = torch.arange(K * d * nnz, dtype=torch.float64).reshape(K, d, nnz) * 0.5
    ref_0 = torch.arange(K * n * n, dtype=torch.float64).reshape(K, n, n) * 0.25
    b = torch.full_like(ref_b, -1.0); A = torch.full_like(ref_A, -1.0); A0 = torch.full_like(ref_0, -1.0)
    lo, hi = ranges[rank]
    b[:, :, lo:hi] = ref_b[:, :, lo:hi]
    A[:, :, row_ptr[lo]:row_ptr[hi]] = ref_A[:, :, row_ptr[lo]:row_ptr[hi]]
    A0[:, lo:hi] = ref_0[:, lo:hi]
    replicate_rows(b, A, A0, row_ptr, ranges, rank)
    q.put((rank, bool(torch.equal(b, ref_b) and torch.equal(A, ref_A) and torch.equal(A0, ref_0))))
    dist.destroy_process_group()


def test_gloo_world2_row_replication_bitwise():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in out), out
