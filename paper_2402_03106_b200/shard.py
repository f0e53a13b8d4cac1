"""Multi-GPU plumbing of the DARTS render.

Paths are independent.  Rank r of n renders the samples
[floor(r S / n), floor((r + 1) S / n)) of every cell (or pixel); since the
Philox counter of a path is its GLOBAL identity (s, p, b), the ranks' key
ranges are disjoint and their union is exactly the one-GPU render.  The one
exchange step is the sum of the per-rank histograms: ONE reduce (NCCL on the
GPU box, gloo in the CPU tests).  No arithmetic of the method lives here.
"""
from __future__ import annotations

from typing import Callable


def shard_range(spp: int, rank: int, world: int) -> tuple[int, int]:
    """Sample range [begin, end) of ``rank`` out of ``world``: contiguous,
    disjoint, covering [0, spp), sizes differing by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if spp < 0:
        raise ValueError("spp must be >= 0")
    return spp * rank // world, spp * (rank + 1) // world


def render_sharded(render_range: Callable[[int, int], None], spp: int, hist, counters=None, dst: int = 0):
    """Renders this rank's sample range with ``render_range(begin, end)`` (which
    must ACCUMULATE into ``hist`` / ``counters``) and then sums the histograms
    onto rank ``dst`` with one reduce, the counters onto every rank.  Works for
    any initialised torch.distributed backend; a no-op exchange at world 1."""
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    b, e = shard_range(spp, rank, world)
    render_range(b, e)
    if world > 1:
        dist.reduce(hist, dst=dst)
        if counters is not None:
            dist.all_reduce(counters)
    return b, e
