#!/usr/bin/env python
"""The sensor-response experiment of PAPER.md:302-310 (Fig. 6) on a synthetic
scene: config 4's cube with walls and two emitters, a 3..9
window of 120 bins and a two-peak tabulated W(t) (dts_inputs.response_config).

Reports, for GPU DARTS (bins drawn ~ W, R31) and GPU vanilla (connections
weighted by W at their arrival time):
  - the fraction of path samples rejected because W = 0 at their time
    (paper: vanilla 85.31 %, DARTS < 3 %);
  - the MSE of the W-weighted image (sum over bins) against a 64x-spp DARTS
    reference at equal render time (CUDA events).
Writes gpurun_out/response_experiment.json.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--crop", type=int, default=512)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--ref-mult", type=int, default=64)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "response_experiment.json"))
    args = ap.parse_args()
    import torch

    from paper_2402_03106_b200 import dts
    c = I.crop_center(I.as_f32(I.response_config()), args.crop, args.crop)
    c["response"] = I.two_peak_response(c["n_bins"], c["t0"], c["t1"])
    spp = c["spp"]
    ref = None
    for k in range(args.ref_mult):
        h, _, _ = _render(dts, torch, c, spp, 10_000 + k)
        ref = h if ref is None else ref + h
    ref /= args.ref_mult
    ref_img = ref.sum(-1)
    out = {"config": c["name"], "crop": c["crop"], "n_bins": c["n_bins"], "spp": spp,
           "response_nonzero_bins": int((np.asarray(c["response"]) > 0).sum()), "strategies": {}}
    _, ms_d0, _ = _render(dts, torch, c, spp, 1)
    for strat in ("darts", "vanilla"):
        cs = dict(c, strategy=strat)
        if strat == "darts":
            sk = spp
        else:
            _, ms0, _ = _render(dts, torch, cs, spp, 2)
            sk = max(1, int(round(spp * ms_d0 / max(ms0, 1e-3))))
        reps = []
        for r in range(args.reps):
            h, ms, cnt = _render(dts, torch, cs, sk, 100 + r)
            reps.append({"ms": ms, "mse_image": float(((h.sum(-1) - ref_img) ** 2).mean()),
                         "mse_hist": float(((h - ref) ** 2).mean()), "samples": cnt["samples"],
                         "rejected": cnt["rejected"], "paths": cnt["paths"]})
        smp = sum(x["samples"] for x in reps)
        rej = sum(x["rejected"] for x in reps)
        out["strategies"][strat] = {
            "spp": sk, "ms": float(np.mean([x["ms"] for x in reps])),
            "mse_image": float(np.mean([x["mse_image"] for x in reps])),
            "mse_image_median": float(np.median([x["mse_image"] for x in reps])),
            "mse_hist": float(np.mean([x["mse_hist"] for x in reps])),
            "rejected_fraction": rej / max(1, smp), "samples": smp, "rejected": rej, "reps": reps}
    d, v = out["strategies"]["darts"], out["strategies"]["vanilla"]
    out["image_mse_ratio_vanilla_over_darts_time_adjusted"] = (v["mse_image"] * v["ms"]) / (d["mse_image"] * d["ms"])
    out["image_median_mse_ratio_vanilla_over_darts_time_adjusted"] = (v["mse_image_median"] * v["ms"]) / (
        d["mse_image_median"] * d["ms"])
    print(json.dumps({k: out[k] for k in ("config", "crop", "response_nonzero_bins",
                                          "image_mse_ratio_vanilla_over_darts_time_adjusted",
                                          "image_median_mse_ratio_vanilla_over_darts_time_adjusted")}))
    for k, s in out["strategies"].items():
        print(f"{k}: spp {s['spp']} {s['ms']:.2f} ms  rejected {100 * s['rejected_fraction']:.2f} % of "
              f"{s['samples']} path samples  image MSE {s['mse_image']:.3e}")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
