#!/usr/bin/env python
"""Small renders of every kernel variant for compute-sanitizer runs:
DARTS (deferred queue, smem table via TMA bulk copy, privatised histogram for
config 1, plain-RED splats), the ablations, RESPONSE mode, vanilla, the
global-memory table path, and dts_sample_debug."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import dts_inputs as I  # noqa: E402
from paper_2402_03106_b200 import dts  # noqa: E402

cases = [
    I.config(1, spp=16),
    I.small(I.config(2), 8, 8),
    I.small(I.config(3), 8, 8, n_bins=32, t1=8.0),
    I.small(I.config(4), 16, 16),
    I.small(I.config(5), 8, 8, n_bins=50, t1=10.0),
    I.config(5, crop=(500, 500, 532, 508), n_bins=200, t1=30.0, spp=8),
    I.small(I.config(4, strategy="eda_only"), 8, 8),
    I.small(I.config(3, strategy="da_only", conn_sampling="uniform"), 8, 8, n_bins=32, t1=8.0),
    I.small(I.config(4, strategy="vanilla"), 16, 16),
    I.config(4, crop=(256, 256, 260, 260), table_nr=32, table_ns=32),
    # camera-ray culling + the start stage (sphere, unwarped camera; meshes), the
    # two-stage render in a sphere, per-pixel mode with culled pixels
    I.config(2, n_bins=32, t1=10.0, spp=4),
    I.small(I.config(6), 24, 24),
    I.config(2, n_bins=32, t1=10.0, spp=4, direction_mode="split"),
    I.config(2, n_bins=32, t1=10.0, spp=64, spp_mode="pixel"),
]
for c in cases:
    c = I.as_f32(c)
    sc = dts.Scene(c)
    if c["strategy"] != "vanilla":
        sc.table_build()
    spp = min(c["spp"], 16)
    h, hs, ctr = dts.render_to_tensor(sc, spp, 1, with_sq=False)
    h2, hs2, _ = dts.render_to_tensor(sc, spp, 1, with_sq=True)
    torch.cuda.synchronize()
    if c["strategy"] != "vanilla":
        out = dts.debug(sc, I.debug_records(c, 64, seed=3))
    print(c["name"], c["strategy"], float(h.sum()), dts.counters_dict(ctr)["vertices"], flush=True)
r = I.small(I.as_f32(I.response_config()), 8, 8)
r["response"] = I.two_peak_response(r["n_bins"], r["t0"], r["t1"])
for st in ("darts", "vanilla"):
    sc = dts.Scene(dict(r, strategy=st))
    sc.table_build()
    h, _, ctr = dts.render_to_tensor(sc, 8, 1)
    torch.cuda.synchronize()
    print("response", st, float(h.sum()), dts.counters_dict(ctr)["samples"], flush=True)
nf = dts.check_failures()
print(f"sanitize cases done; device bounds-check failures: {nf}")
sys.exit(1 if nf else 0)
