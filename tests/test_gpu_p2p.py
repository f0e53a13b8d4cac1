"""Fused render + reduce through peer memory (paper_2402_03106_b200.shard.
render_sharded_p2p): two processes render disjoint Philox sample ranges, the
second one straight into the first one's histogram through a CUDA IPC mapping
(NVLink peer memory on a multi-GPU box; here both processes share cuda:0, which
exercises the same mapping and cross-process REDs -- the kernels never wait on
one another).  The result equals the one-process render up to fp32 summation
order."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import dts_inputs as I

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, c, spp, seed, out):
    import torch.distributed as dist

    from paper_2402_03106_b200 import dts
    from paper_2402_03106_b200.shard import release_peer_histograms, render_sharded_p2p
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = dts.Scene(c)
    sc.table_build()
    hist = torch.zeros(sc.hist_shape(), dtype=torch.float32, device="cuda")
    ctr = torch.zeros(dts.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    for step in range(2):   # the second step reuses the mapping and re-zeroes rank 0's histogram
        c_step = torch.zeros_like(ctr)
        render_sharded_p2p(lambda b, e, t: sc.render(spp, seed, b, e, t, None, c_step), spp, hist, c_step.cpu(),
                           enable_peer=dts.enable_peer)
    if rank == 0:
        np.save(out, hist.cpu().numpy())
    release_peer_histograms()
    torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()


def test_p2p_fused_reduce_equals_single_render(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp

    from paper_2402_03106_b200 import dts
    c = I.as_f32(I.small(I.config(3), 16, 16, n_bins=64, t1=9.0))
    spp, seed = 24, 5
    out = str(tmp_path / "h.npy")
    mp.spawn(_worker, args=(2, _free_port(), c, spp, seed, out), nprocs=2, join=True)
    got = np.load(out)
    sc = dts.Scene(c)
    sc.table_build()
    ref, _, _ = dts.render_to_tensor(sc, spp, seed)
    ref = ref.cpu().numpy()
    assert np.count_nonzero(ref) > 100
    assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref)
