"""Multi-GPU batch sharding (config 4).

Images are independent problems (the reference is reentrant), so
a batch shards across ranks with no data-path collective: every rank solves
the images of its LPT shard on its own GPU (one process per GPU, launched by
torchrun) and only the timing is reduced (max over ranks, on the device
clock).  A single large image is NOT split across GPUs here: exact
Gauss-Seidel order makes that a pipelined cross-GPU wavefront (DESIGN.md,
"Multi-GPU"), not a halo exchange.
"""
from __future__ import annotations

import heapq
from typing import List, Sequence, Tuple


def lpt_partition(sizes: Sequence[Tuple[int, int]], nranks: int) -> List[List[int]]:
    """Longest-processing-time partition of image indices by pixel count.
    Deterministic: ties broken by index, so every rank computes the same
    partition without communication."""
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    order = sorted(range(len(sizes)), key=lambda i: (-sizes[i][0] * sizes[i][1], i))
    heap = [(0, r) for r in range(nranks)]
    shards: List[List[int]] = [[] for _ in range(nranks)]
    for i in order:
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + sizes[i][0] * sizes[i][1], r))
    for s in shards:
        s.sort()
    return shards


def shard_pixels(sizes, shard) -> int:
    return sum(sizes[i][0] * sizes[i][1] for i in shard)


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank scalar (the timed region's device
    milliseconds); identity when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
