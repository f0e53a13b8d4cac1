#!/usr/bin/env python
"""Equal-time MSE of GPU DARTS vs the GPU vanilla baseline (same kernels,
north_star "MSE vs oracle at equal time").

Per config (a centre crop for the large ones):
  1. reference = GPU DARTS at ref_mult x the config's spp (independent seeds);
  2. DARTS at the config's spp: device time T (CUDA events) and MSE vs the reference;
  3. vanilla with its spp calibrated so its render takes ~T, MSE vs the reference;
  4. repeated over `reps` seeds; MSE normalised to DARTS = 1.
For configs 3 and 5 both direction modes (REUSE, SPLIT) are measured (R29).
Writes gpurun_out/mse_equal_time.json.

    python scripts/mse_equal_time.py [--configs 1 2 3 4 5] [--reps 4]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import dts_inputs as I  # noqa: E402

CROPS = {1: None, 2: None, 3: 32, 4: 128, 5: 32}


def _render(dts, torch, c, spp, seed):
    sc = dts.Scene(c)
    if c["strategy"] == "darts":
        sc.table_build()
    h = torch.zeros(sc.hist_shape(), dtype=torch.float32, device="cuda")
    ctr = torch.zeros(dts.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sc.render(spp, seed, 0, spp, h, None, ctr)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    sc.close()
    return h.double(), ms, dts.counters_dict(ctr)


def run_config(dts, torch, idx, mode, reps, ref_mult):
    c = I.as_f32(I.config(idx, direction_mode=mode))
    if CROPS[idx]:
        c = I.crop_center(c, CROPS[idx], CROPS[idx])
    spp = c["spp"]
    # reference: ref_mult x spp, rendered in chunks of spp with distinct seeds
    ref = None
    for k in range(ref_mult):
        h, _, _ = _render(dts, torch, c, spp, 10_000 + k)
        ref = h if ref is None else ref + h
    ref /= ref_mult
    out = {"config": idx, "mode": mode, "crop": c["crop"], "spp": spp, "ref_mult": ref_mult, "reps": []}
    cv = dict(c, strategy="vanilla")
    # vanilla spp per pixel: start at the DARTS paths per pixel, calibrate on time
    paths_px = spp * (c["n_bins"] if c["spp_mode"] == "cell" else 1)
    _, ms_d0, _ = _render(dts, torch, c, spp, 1)
    _, ms_v0, _ = _render(dts, torch, cv, paths_px, 2)
    spp_v = max(1, int(round(paths_px * ms_d0 / max(ms_v0, 1e-3))))
    for r in range(reps):
        hd, ms_d, cd = _render(dts, torch, c, spp, 100 + r)
        hv, ms_v, cvv = _render(dts, torch, cv, spp_v, 200 + r)
        mse_d = float(((hd - ref) ** 2).mean())
        mse_v = float(((hv - ref) ** 2).mean())
        out["reps"].append({"ms_darts": ms_d, "ms_vanilla": ms_v, "mse_darts": mse_d, "mse_vanilla": mse_v,
                            "vertices_darts": cd["vertices"], "vertices_vanilla": cvv["vertices"]})
    ms_d = np.mean([x["ms_darts"] for x in out["reps"]])
    ms_v = np.mean([x["ms_vanilla"] for x in out["reps"]])
    md = np.mean([x["mse_darts"] for x in out["reps"]])
    mv = np.mean([x["mse_vanilla"] for x in out["reps"]])
    out.update({"spp_vanilla_per_pixel": spp_v, "ms_darts": ms_d, "ms_vanilla": ms_v, "mse_darts": md,
                "mse_vanilla": mv, "mse_ratio_vanilla_over_darts": mv / md if md > 0 else None,
                "equal_time_mse_ratio": (mv * ms_v) / (md * ms_d) if md > 0 else None,
                "ref_signal_ms": float((ref ** 2).mean())})
    print(f"cfg{idx}/{mode}: DARTS {ms_d:.1f} ms MSE {md:.3e} | vanilla spp {spp_v} {ms_v:.1f} ms MSE {mv:.3e} "
          f"| ratio {out['mse_ratio_vanilla_over_darts']:.2f} (time-adjusted {out['equal_time_mse_ratio']:.2f})",
          flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--ref-mult", type=int, default=64)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "mse_equal_time.json"))
    args = ap.parse_args()
    import torch

    from paper_2402_03106_b200 import dts
    res = []
    for idx in args.configs:
        modes = ["reuse", "split"] if idx in (3, 5) else [I.config(idx)["direction_mode"]]
        for m in modes:
            res.append(run_config(dts, torch, idx, m, args.reps, args.ref_mult))
            os.makedirs(os.path.dirname(args.out), exist_ok=True)
            with open(args.out, "w") as f:
                json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
