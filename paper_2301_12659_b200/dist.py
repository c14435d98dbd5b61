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
