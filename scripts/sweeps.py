#!/usr/bin/env python
"""Scattering-coefficient and gate-width sweeps (the setting of
PAPER.md:376-417, Figs. 9-10) on the config-3 slab: a single time gate, GPU
DARTS vs the GPU vanilla baseline at equal render time, MSE of the gated image
against a 64x-spp DARTS reference, normalised by the reference's mean square
(relative MSE) -- and, as the paper does, also by DARTS's own MSE.

  sigma_s sweep : sigma_s in {2, 4, 6, 8, 10, 12}, sigma_a 0.1, g 0.8, gate [6.0, 6.1)
  gate sweep    : sigma_s 9.9, gate [6.0, 6.0 + w), w in {0.025, 0.05, 0.1, 0.2, 0.4, 0.8}
Writes gpurun_out/sweeps.json.
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


def _render(dts, torch, c, spp, seed):
    sc = dts.Scene(c)
    if c["strategy"] != "vanilla":
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
    return h.double(), ms


def point(dts, torch, c, spp, reps, ref_mult):
    ref = None
    for k in range(ref_mult):
        h, _ = _render(dts, torch, c, spp, 10_000 + k)
        ref = h if ref is None else ref + h
    ref /= ref_mult
    norm = float((ref ** 2).mean())
    _, ms_d0 = _render(dts, torch, c, spp, 1)
    cv = dict(c, strategy="vanilla")
    _, ms_v0 = _render(dts, torch, cv, spp, 2)
    spp_v = max(1, int(round(spp * ms_d0 / max(ms_v0, 1e-3))))
    res = {}
    for name, cs, sk in (("darts", c, spp), ("vanilla", cv, spp_v)):
        mses, mss = [], []
        for r in range(reps):
            h, ms = _render(dts, torch, cs, sk, 100 + r)
            mses.append(float(((h - ref) ** 2).mean()))
            mss.append(ms)
        res[name] = {"spp": sk, "ms": float(np.mean(mss)), "rel_mse": float(np.mean(mses)) / norm,
                     "rel_mse_median": float(np.median(mses)) / norm}
    res["vanilla_over_darts_time_adjusted"] = (res["vanilla"]["rel_mse"] * res["vanilla"]["ms"]) / (
        res["darts"]["rel_mse"] * res["darts"]["ms"])
    res["vanilla_over_darts_median_time_adjusted"] = (res["vanilla"]["rel_mse_median"] * res["vanilla"]["ms"]) / (
        res["darts"]["rel_mse_median"] * res["darts"]["ms"])
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--crop", type=int, default=64)
    ap.add_argument("--spp", type=int, default=256)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--ref-mult", type=int, default=64)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweeps.json"))
    args = ap.parse_args()
    import torch

    from paper_2402_03106_b200 import dts
    out = {"sigma_s": [], "gate": [], "crop": args.crop, "spp": args.spp}
    for ss in (2.0, 4.0, 6.0, 8.0, 10.0, 12.0):
        c = I.as_f32(I.config(3, sigma_s=ss, t0=6.0, t1=6.1, n_bins=1, spp=args.spp))
        c = I.crop_center(c, args.crop, args.crop)
        r = point(dts, torch, c, args.spp, args.reps, args.ref_mult)
        r["sigma_s"] = ss
        out["sigma_s"].append(r)
        print(f"sigma_s {ss:5.1f}: DARTS rel MSE {r['darts']['rel_mse']:.3e} ({r['darts']['ms']:.2f} ms) | vanilla "
              f"{r['vanilla']['rel_mse']:.3e} ({r['vanilla']['ms']:.2f} ms, spp {r['vanilla']['spp']}) | "
              f"vanilla/DARTS x time {r['vanilla_over_darts_time_adjusted']:.2f} (median {r['vanilla_over_darts_median_time_adjusted']:.2f})", flush=True)
    for w in (0.025, 0.05, 0.1, 0.2, 0.4, 0.8):
        c = I.as_f32(I.config(3, t0=6.0, t1=6.0 + w, n_bins=1, spp=args.spp))
        c = I.crop_center(c, args.crop, args.crop)
        r = point(dts, torch, c, args.spp, args.reps, args.ref_mult)
        r["gate_width"] = w
        out["gate"].append(r)
        print(f"gate {w:6.3f}: DARTS rel MSE {r['darts']['rel_mse']:.3e} ({r['darts']['ms']:.2f} ms) | vanilla "
              f"{r['vanilla']['rel_mse']:.3e} ({r['vanilla']['ms']:.2f} ms, spp {r['vanilla']['spp']}) | "
              f"vanilla/DARTS x time {r['vanilla_over_darts_time_adjusted']:.2f} (median {r['vanilla_over_darts_median_time_adjusted']:.2f})", flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
