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
