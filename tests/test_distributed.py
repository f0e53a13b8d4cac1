"""Multi-process (world size 2, gloo, CPU) test of the sharded render's host
logic: disjoint sample ranges + one reduce reproduce the
single-process render.  The per-rank renders are the fp64 oracle (this is the
CPU stand-in for libdts on a GPU box); the sharding and reduce code is the
product's own ``paper_2402_03106_b200.shard``."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import dts_inputs as I  # noqa: E402
from paper_2402_03106_b200.shard import render_sharded, shard_range  # noqa: E402


def test_shard_ranges_partition():
    for spp in (0, 1, 7, 1024):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(spp, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == spp
            for (a, b), (c, d) in zip(rs, rs[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, spp, seed, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    c = cfg
    q = O.build_table(c, nthreads=1)[0] if c["strategy"] == "darts" else None
    hist = torch.zeros(I.n_cells(c), dtype=torch.float64)
    ctr = torch.zeros(2, dtype=torch.int64)

    def render_range(b, e):
        r = O.render(c, q, spp, seed, s_begin=b, s_end=e, sq=False, nthreads=1)
        hist.add_(torch.from_numpy(r["hist"].ravel()))
        ctr.add_(torch.tensor([r["stats"]["paths"], r["stats"]["vertices"]], dtype=torch.int64))

    render_sharded(render_range, spp, hist, ctr)
    if rank == 0:
        np.save(out_path, np.concatenate([hist.numpy(), ctr.numpy().astype(np.float64)]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg_name", ["cfg4_small", "cfg5_pixelmode"])
def test_two_rank_gloo_reduce_equals_single_render(tmp_path, cfg_name):
    from oracle import oracle as O
    if cfg_name == "cfg4_small":
        c, spp = I.as_f32(I.small(I.config(4), 6, 6)), 9
    else:
        c, spp = I.as_f32(I.small(I.config(5), 3, 3, n_bins=40, t1=8.0)), 40
    seed = 11
    out = str(tmp_path / "h.npy")
    mp.spawn(_worker, args=(2, _free_port(), c, spp, seed, out), nprocs=2, join=True)
    got = np.load(out)
    n = I.n_cells(c)
    q = O.build_table(c)[0]
    ref = O.render(c, q, spp, seed, sq=False)
    h = ref["hist"].ravel()
    assert np.linalg.norm(got[:n] - h) <= 1e-12 * max(np.linalg.norm(h), 1e-300)
    assert int(got[n]) == ref["stats"]["paths"] and int(got[n + 1]) == ref["stats"]["vertices"]
    assert np.count_nonzero(h) > 0


def _band_worker(rank, world, port, cfg, spp, seed, nbands, out_path):
    """bench.py's end-to-end pipeline at N ranks (shard.pipeline_bands), with the
    fp64 oracle rendering each rank's sample range of a row band in place of
    dts_render_rows: band renders, gloo reduces onto rank 0 in band order, and
    rank 0's copies into its host array."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2402_03106_b200.shard import pipeline_bands
    c = cfg
    q = O.build_table(c, nthreads=1)[0]
    x0, y0, x1, y1 = c["crop"]
    rowsz = (x1 - x0) * c["n_bins"]
    dev = torch.zeros((y1 - y0) * rowsz, dtype=torch.float64)
    host = np.full(dev.numel(), np.nan) if rank == 0 else None
    b, e = shard_range(spp, rank, world)
    order = []

    def render_rows(k, r0, r1):
        cb = dict(c, crop=(x0, y0 + r0, x1, y0 + r1))
        r = O.render(cb, q, spp, seed, s_begin=b, s_end=e, sq=False, nthreads=1)
        dev[r0 * rowsz:r1 * rowsz] += torch.from_numpy(r["hist"].ravel())
        order.append(("render", k))

    def reduce_band(k, r0, r1):
        band = dev[r0 * rowsz:r1 * rowsz].clone()
        dist.reduce(band, dst=0)
        if rank == 0:
            dev[r0 * rowsz:r1 * rowsz] = band
        order.append(("reduce", k))

    def to_host(k, r0, r1):
        host[r0 * rowsz:r1 * rowsz] = dev[r0 * rowsz:r1 * rowsz].numpy()
        order.append(("copy", k))

    pipeline_bands(y1 - y0, nbands, render_rows, reduce_band, to_host, world, rank)
    if rank == 0:
        np.save(out_path, host)
        # per band: render, reduce, copy; bands in order
        exp = [(s, k) for k in range(nbands) for s in ("render", "reduce", "copy")]
        assert order == exp, order
    else:
        assert order == [(s, k) for k in range(nbands) for s in ("render", "reduce")], order
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_banded_e2e_pipeline_equals_single_render(tmp_path):
    """The banded render / reduce / host-copy pipeline of bench.py's e2e leg at
    N = 2 (gloo): the host histogram rank 0 assembles band by band equals the
    single-process full render, every band is reduced in the same order on every
    rank, and bands are contiguous and complete (shard.band_rows)."""
    from oracle import oracle as O
    from paper_2402_03106_b200.shard import band_rows
    c, spp, seed, nbands = I.as_f32(I.small(I.config(5), 5, 9, n_bins=30, t1=9.0)), 12, 7, 4
    out = str(tmp_path / "host.npy")
    mp.spawn(_band_worker, args=(2, _free_port(), c, spp, seed, nbands, out), nprocs=2, join=True)
    got = np.load(out)
    assert np.isfinite(got).all()
    ref = O.render(c, O.build_table(c)[0], spp, seed, sq=False)["hist"].ravel()
    assert np.count_nonzero(ref) > 0
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    assert band_rows(9, 4) == [(0, 2), (2, 5), (5, 8), (8, 9)]
    assert band_rows(1024, 4)[-1] == (992, 1024) and band_rows(10, 1) == [(0, 10)]
    with pytest.raises(ValueError):
        band_rows(3, 4)
