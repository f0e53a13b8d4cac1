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


def band_rows(rows: int, nbands: int) -> list[tuple[int, int]]:
    """Row bands [r0, r1) of a crop of ``rows`` rows: contiguous and covering;
    with more than one band the last is short (1/32 of the rows, at least one
    row) -- only its host copy is not hidden behind a later band's render -- and
    the others split the rest within one row (dts_render_host does the same)."""
    if nbands < 1 or rows < 2 * nbands:
        raise ValueError(f"need 1 <= nbands <= rows / 2, got {nbands} bands of {rows} rows")
    if nbands == 1:
        return [(0, rows)]
    cut = rows - max(1, rows // 32)
    m = nbands - 1
    return [(cut * k // m, cut * (k + 1) // m) for k in range(m)] + [(cut, rows)]


def pipeline_bands(rows: int, nbands: int, render_rows: Callable[[int, int, int], None],
                   reduce_band: Callable[[int, int, int], None], to_host: Callable[[int, int, int], None],
                   world: int, rank: int, dst: int = 0) -> None:
    """The end-to-end pipeline of a large histogram at N ranks:
    band by band, every rank renders its sample range of the band
    (``render_rows(k, r0, r1)``), the band is reduced onto rank ``dst``
    (``reduce_band``: a collective, issued in the same band order on every rank),
    and rank ``dst`` starts the band's copy to the host (``to_host``, e.g. on a
    copy stream) while the next band renders.  No arithmetic of the method here."""
    for k, (r0, r1) in enumerate(band_rows(rows, nbands)):
        render_rows(k, r0, r1)
        if world > 1:
            reduce_band(k, r0, r1)
        if rank == dst:
            to_host(k, r0, r1)


_PEER_CACHE: dict = {}


def peer_histogram(hist, dst: int = 0, enable_peer: Callable[[int], None] | None = None):
    """The histogram every rank renders into for the fused reduce: rank dst's
    own tensor there, elsewhere the same device memory mapped through CUDA IPC
    (peer memory over NVLink / NVSwitch on a multi-GPU box).  Collective: the
    cache key is rank dst's (address, size), broadcast on every call, so all
    ranks hit or miss together; a mapping is opened once per key.
    ``enable_peer(device)`` (libdts' dts_enable_peer) is called with the device
    that owns the mapping, so that this rank's kernels may access it."""
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor

    me = dist.get_rank()
    hdr = [(hist.data_ptr(), hist.numel(), hist.device.index) if me == dst else None]
    dist.broadcast_object_list(hdr, src=dst)
    key = (hdr[0], dst)
    hit = [key in _PEER_CACHE]
    # every rank must agree on hit / miss before the (collective) mapping step
    flags = [None] * dist.get_world_size()
    dist.all_gather_object(flags, hit[0])
    if all(flags):
        return _PEER_CACHE[key]
    obj = [reduce_tensor(hist) if me == dst else None]
    dist.broadcast_object_list(obj, src=dst)
    if me == dst:
        target = hist
    else:
        fn, args = obj[0]
        target = fn(*args)
        if enable_peer is not None and target.device.index is not None:
            enable_peer(target.device.index)
    _PEER_CACHE[key] = target
    return target


def release_peer_histograms() -> None:
    """Drops this process's peer mappings (before the producer rank exits)."""
    _PEER_CACHE.clear()


def render_sharded_p2p(render_range: Callable, spp: int, hist, counters=None, dst: int = 0, zero: bool = True,
                       enable_peer: Callable[[int], None] | None = None):
    """Fused render + reduce: each rank's render kernel adds its contributions
    (fp32 REDs) directly into rank dst's histogram through peer memory, so no
    reduce collective follows -- the transfer overlaps the render path by path.
    ``render_range(begin, end, target)`` must render into ``target``.  With
    ``zero`` rank dst clears its histogram first (every rank waits for it).
    rank dst's ``hist`` holds the sum when this returns (every rank synchronises
    and meets at a barrier); the other ranks' ``hist`` are untouched.
    EXPERIMENTAL: checked with two processes on one GPU only (the pool has one
    GPU per call); NCCL's reduce stays the default until a multi-GPU run."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    b, e = shard_range(spp, rank, world)
    target = hist if world == 1 else peer_histogram(hist, dst, enable_peer)
    if zero and rank == dst:
        hist.zero_()
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
    render_range(b, e, target)
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
        if counters is not None:
            dist.all_reduce(counters)
    return b, e
