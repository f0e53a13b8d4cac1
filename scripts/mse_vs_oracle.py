#!/usr/bin/env python
"""MSE of GPU DARTS vs the CPU oracle at equal time (BASELINE.json metric
"MSE vs oracle at equal time") on a config-5 crop.

1. The fp64 oracle renders a centre crop (all bins, the config's spp) on all
   host cores: wall time T_cpu, histogram h_cpu.
2. A GPU reference at ref_mult x spp (same estimator, independent seeds).
3. GPU renders of the crop at spp x {1, 4, 16, 64} (several seeds each):
   device time and MSE vs the reference -> the MSE(spp) slope (variance
   scaling: MSE ~ 1/spp) and the GPU's MSE at the oracle's spp.
4. Equal time: the GPU sample count the oracle's T_cpu buys is T_cpu / T_gpu(spp)
   x spp; its MSE is read off the measured power law (stated as an
   extrapolation where it exceeds the largest measured spp).
Writes gpurun_out/mse_vs_oracle.json.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import dts_inputs as I  # noqa: E402


def gpu_render(dts, torch, c, spp, seed):
    sc = dts.Scene(c)
    sc.table_build()
    h = torch.zeros(sc.hist_shape(), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sc.render(spp, seed, 0, spp, h)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    sc.close()
    return h.double().cpu().numpy(), ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--crop", type=int, default=16)
    ap.add_argument("--ref-mult", type=int, default=256)
    ap.add_argument("--seeds", type=int, default=6)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "mse_vs_oracle.json"))
    args = ap.parse_args()
    import torch

    from oracle import oracle as O
    from paper_2402_03106_b200 import dts
    c = I.crop_center(I.as_f32(I.config(args.config)), args.crop, args.crop)
    spp = c["spp"]
    q = O.build_table(c)[0]
    t = time.perf_counter()
    o = O.render(c, q, spp, 77, sq=False, nthreads=os.cpu_count())
    t_cpu = time.perf_counter() - t
    h_cpu = o["hist"]
    ref = None
    for k in range(args.ref_mult // 16):
        h, _ = gpu_render(dts, torch, c, spp * 16, 20_000 + k)
        ref = h if ref is None else ref + h
    ref /= args.ref_mult // 16
    mse_cpu = float(((h_cpu - ref) ** 2).mean())
    pts = []
    for mult in (1, 4, 16, 64):
        if mult * 4 > args.ref_mult:
            break
        ms, mse = [], []
        for s in range(args.seeds):
            h, m = gpu_render(dts, torch, c, spp * mult, 100 * mult + s)
            ms.append(m)
            mse.append(float(((h - ref) ** 2).mean()))
        # (the reference's own error, ~ MSE(spp) spp / (ref_mult spp_ref), is not subtracted)
        pts.append({"spp": spp * mult, "ms": float(np.median(ms)), "mse": float(np.mean(mse))})
    x = np.log([p["spp"] for p in pts])
    y = np.log([p["mse"] for p in pts])
    slope, icpt = np.polyfit(x, y, 1)
    g1 = pts[0]
    gl = pts[-1]  # the largest launch: the GPU's steady-state throughput on this crop
    spp_eq = gl["spp"] * t_cpu * 1e3 / gl["ms"]
    mse_gpu_eq = float(np.exp(icpt + slope * np.log(spp_eq)))
    out = {"config": c["name"], "crop": c["crop"], "spp": spp, "cpu_cores": os.cpu_count(), "t_cpu_s": t_cpu,
           "oracle_vertices": o["stats"]["vertices"], "mse_cpu": mse_cpu, "gpu_points": pts,
           "mse_vs_spp_slope": float(slope), "gpu_spp_at_equal_time": spp_eq,
           "gpu_mse_at_equal_time_powerlaw": mse_gpu_eq, "mse_ratio_cpu_over_gpu_equal_time": mse_cpu / mse_gpu_eq,
           "mse_ratio_cpu_over_gpu_equal_spp": mse_cpu / g1["mse"],
           "note": "equal-time GPU MSE read off the measured MSE(spp) power law; extrapolated beyond the largest "
                   "measured spp; the reference's own error (~1/ref_mult of MSE(spp)) is not subtracted"}
    print(json.dumps({k: v for k, v in out.items() if k != "gpu_points"}))
    for p in pts:
        print(f"GPU spp {p['spp']}: {p['ms']:.2f} ms  MSE {p['mse']:.3e}")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
