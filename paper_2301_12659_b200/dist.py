"""Multi-GPU plumbing for the batched path.

Paths are independent units: rank r of N owns the contiguous path range
``partition(batch, N, r)`` and runs ``ns_newton_series_step_batched`` on it.
There is no collective in the step.  torch.distributed (NCCL on GPUs, gloo in
the CPU tests) is used only for the host-side plumbing around it: a barrier,
the max over ranks of the timed region, and an optional all-gather of the
per-path residual norms for reporting.
"""
from __future__ import annotations


def partition(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split of `batch` paths: the first batch % world ranks
    get one extra path.  Returns [lo, hi)."""
    if world < 1 or not (0 <= rank < world) or batch < 0:
        raise ValueError("bad partition arguments")
    q, r = divmod(batch, world)
    lo = rank * q + min(rank, r)
    hi = lo + q + (1 if rank < r else 0)
    return lo, hi


def max_over_ranks(value: float, device=None) -> float:
    """Max of a float over all ranks (the timing rule: slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def gather_paths(local, batch: int, device=None):
    """All-gather per-path tensors (first dim = local paths, contiguous ranges
    from `partition`) into one [batch, ...] tensor on every rank; pads the
    uneven shares (all_gather needs equal sizes)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    q = -(-batch // world)
    pad = torch.zeros((q,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    parts = []
    for r in range(world):
        lo, hi = partition(batch, world, r)
        parts.append(bufs[r][:hi - lo])
    return torch.cat(parts, 0)


# ------------------------------------------------------------------ C4: sharded eval/diff
def equation_costs(eq_ptr, mono_ptr, d: int):
    """Convolution work of each equation: sum over its monomials of (3m - 5)
    products of d(d+1)/2 multiply-adds (m = 1: 0, m = 2: 1 product) plus the
    m d scaling multiply-adds."""
    tri = d * (d + 1) // 2
    out = []
    for i in range(len(eq_ptr) - 1):
        c = 0
        for t in range(int(eq_ptr[i]), int(eq_ptr[i + 1])):
            m = int(mono_ptr[t + 1] - mono_ptr[t])
            p = 0 if m <= 1 else (1 if m == 2 else 3 * m - 5)
            c += p * tri + (m + 1) * d
        out.append(c)
    return out


def equation_partition(eq_ptr, mono_ptr, d: int, world: int):
    """Contiguous equation ranges, one per rank, balanced by the prefix sum of
    the equation costs (equation-owner sharding: no arithmetic reduction is
    needed)."""
    costs = equation_costs(eq_ptr, mono_ptr, d)
    n = len(costs)
    if world > n:
        raise ValueError("more ranks than equations")
    total = sum(costs)
    bounds = [0]
    acc = 0
    r = 1
    for i, c in enumerate(costs):
        acc += c
        # close the current range once its share is reached, leaving enough rows for the rest
        while r < world and acc >= total * r / world and (i + 1) > bounds[-1] and n - (i + 1) >= world - r:
            bounds.append(i + 1)
            r += 1
    while len(bounds) < world:
        bounds.append(n - (world - len(bounds)))
    bounds.append(n)
    return [(bounds[k], bounds[k + 1]) for k in range(world)]


def _row_slices(row_ptr, lo, hi):
    return int(row_ptr[lo]), int(row_ptr[hi])


def replicate_rows(b, A, A0, row_ptr, ranges, rank: int):
    """Row replication after sharded eval/diff: every rank contributes its
    rows [lo, hi) of b [K][d][n], A [K][d][nnz] (entries row_ptr[lo]..row_ptr[hi])
    and A0 [K][n][n]; one all-gather per array (padded to equal sizes), then
    each rank writes the other ranks' rows in place.  Bitwise: rows are copied,
    never summed (never ncclSum on limb planes)."""
    import torch
    import torch.distributed as dist
    world = len(ranges)
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return b, A, A0
    lo, hi = ranges[rank]
    rmax = max(h - l for l, h in ranges)
    emax = max(int(row_ptr[h]) - int(row_ptr[l]) for l, h in ranges)
    K, d, n = b.shape
    # pack
    pb = torch.zeros((K, d, rmax), dtype=b.dtype, device=b.device)
    pb[:, :, :hi - lo] = b[:, :, lo:hi]
    e0, e1 = _row_slices(row_ptr, lo, hi)
    pA = torch.zeros((K, d, emax), dtype=A.dtype, device=A.device)
    pA[:, :, :e1 - e0] = A[:, :, e0:e1]
    p0 = torch.zeros((K, rmax, n), dtype=A0.dtype, device=A0.device)
    p0[:, :hi - lo, :] = A0[:, lo:hi, :]
    gb = [torch.empty_like(pb) for _ in range(world)]
    gA = [torch.empty_like(pA) for _ in range(world)]
    g0 = [torch.empty_like(p0) for _ in range(world)]
    dist.all_gather(gb, pb)
    dist.all_gather(gA, pA)
    dist.all_gather(g0, p0)
    for r, (l, h) in enumerate(ranges):
        if r == rank:
            continue
        f0, f1 = _row_slices(row_ptr, l, h)
        b[:, :, l:h] = gb[r][:, :, :h - l]
        A[:, :, f0:f1] = gA[r][:, :, :f1 - f0]
        A0[:, l:h, :] = g0[r][:, :h - l, :]
    return b, A, A0
