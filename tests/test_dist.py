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


# ------------------------------------------------------------------ C4: the library's row replication plan
def _c4_like(n=40, w=6, D=5, K=4):
    import synth
    return synth.banded_two_column_system(n, w, D, K, seed=3)


def test_exchange_plan_through_c_abi_matches_partition():
    """ns_exchange_plan (host only, through the C ABI) gives the equation
    ranges of dist.equation_partition and the block sizes of the layout
    contract in include/ns.h: K (d (rows + entries) + rows n)."""
    import numpy as np

    import paper_2301_12659_b200 as P
    from oracle import newton as O
    from paper_2301_12659_b200.dist import equation_partition
    for sys_ in (_c4_like(), _c4_like(64, 32, 31, 4), _c4_like(9, 3, 2, 2)):
        rp = np.cumsum([0] + [len(r) for r in O.jacobian_pattern(sys_)])
        for world in (1, 2, 3, 8):
            if world > sys_.n:
                continue
            b, c = P.exchange_plan(sys_.eq_ptr, sys_.mono_ptr, sys_.var_idx, sys_.n, sys_.D, sys_.K, world)
            ranges = equation_partition(sys_.eq_ptr, sys_.mono_ptr, sys_.d, world)
            assert [(int(b[r]), int(b[r + 1])) for r in range(world)] == ranges
            for r, (lo, hi) in enumerate(ranges):
                assert c[r] == sys_.K * (sys_.d * ((hi - lo) + (rp[hi] - rp[lo])) + (hi - lo) * sys_.n)


def _pack(b, A, A0, rp, lo, hi):
    """the block layout of include/ns.h (ns_exchange_plan), restated in numpy"""
    import numpy as np
    return np.concatenate([b[:, :, lo:hi].reshape(-1), A[:, :, rp[lo]:rp[hi]].reshape(-1), A0[:, lo:hi, :].reshape(-1)])


def _unpack(blk, b, A, A0, rp, lo, hi):
    K, d, n = b.shape
    nb, na = K * d * (hi - lo), K * d * (rp[hi] - rp[lo])
    b[:, :, lo:hi] = blk[:nb].reshape(K, d, hi - lo)
    A[:, :, rp[lo]:rp[hi]] = blk[nb:nb + na].reshape(K, d, rp[hi] - rp[lo])
    A0[:, lo:hi, :] = blk[nb + na:].reshape(K, hi - lo, n)


def _replicate_worker(rank, world, port, q):
    import numpy as np

    import paper_2301_12659_b200 as P
    from oracle import newton as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys_ = _c4_like()
    K, d, n = sys_.K, sys_.d, sys_.n
    rp = np.cumsum([0] + [len(r) for r in O.jacobian_pattern(sys_)])
    rng = np.random.default_rng(17)                       # the same "evaluated" arrays on every rank
    fb, fA, f0 = rng.random((K, d, n)), rng.random((K, d, int(rp[-1]))), rng.random((K, n, n))
    bounds, cnt = P.exchange_plan(sys_.eq_ptr, sys_.mono_ptr, sys_.var_idx, n, sys_.D, K, world)
    off = np.concatenate([[0], np.cumsum(cnt)])
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    b, A, A0 = np.zeros_like(fb), np.zeros_like(fA), np.zeros_like(f0)   # this rank's rows only
    b[:, :, lo:hi], A[:, :, rp[lo]:rp[hi]], A0[:, lo:hi] = fb[:, :, lo:hi], fA[:, :, rp[lo]:rp[hi]], f0[:, lo:hi]
    gather = torch.zeros(int(off[-1]), dtype=torch.float64)
    gather[off[rank]:off[rank + 1]] = torch.from_numpy(_pack(b, A, A0, rp, lo, hi))
    for r in range(world):                                # the grouped broadcast, one root per block
        seg = gather[off[r]:off[r + 1]].clone()
        dist.broadcast(seg, src=r)
        gather[off[r]:off[r + 1]] = seg
    for r in range(world):
        if r != rank:
            _unpack(gather[off[r]:off[r + 1]].numpy(), b, A, A0, rp, int(bounds[r]), int(bounds[r + 1]))
    q.put((rank, bool((b == fb).all() and (A == fA).all() and (A0 == f0).all())))
    dist.destroy_process_group()


def test_gloo_world2_row_replication_plan():
    """The library's exchange (ns_comm_init path) on CPU: the plan from the
    C ABI, each rank's rows packed in the contract layout, one broadcast per
    root block over gloo, unpacked: every rank ends with every row, bitwise."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replicate_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in out), out
