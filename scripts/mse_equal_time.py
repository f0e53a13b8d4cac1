#!/usr/bin/env python
"""Equal-time MSE of GPU DARTS vs its ablations (DA-only, EDA-only,
PAPER.md:426-435), uniform-S elliptical sampling and the GPU
vanilla baseline -- same kernels (north_star "MSE vs oracle at equal time";
SURVEY 8(d.4) (i), 8(f) #1).

Per config (a centre crop for the large ones):
  1. reference = GPU DARTS at ref_mult x the config's spp (independent seeds);
  2. DARTS at the config's spp: device time T (CUDA events) and MSE vs the reference;
  3. every other strategy with its spp calibrated so its render takes ~T;
  4. repeated over `reps` seeds; MSE x time normalised to DARTS = 1.
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

CROPS = {1: None, 2: None, 3: 32, 4: 128, 5: 32, 6: None}


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


def run_config(dts, torch, idx, mode, nreps, ref_mult, strategies):
    c = I.as_f32(I.config(idx, direction_mode=mode))
    if CROPS[idx]:
        c = I.crop_center(c, CROPS[idx], CROPS[idx])
    spp = c["spp"]
    # reference: DARTS in the config's own direction mode (SPLIT for the
    # strongly forward configs 3 and 5, R29) at ref_mult x spp, rendered in
    # chunks of spp with distinct seeds
    cref = dict(c, direction_mode=I.config(idx)["direction_mode"])
    ref = None
    for k in range(ref_mult):
        h, _, _ = _render(dts, torch, cref, spp, 10_000 + k)
        ref = h if ref is None else ref + h
    ref /= ref_mult
    out = {"config": idx, "mode": mode, "crop": c["crop"], "spp": spp, "ref_mult": ref_mult, "strategies": {}}
    # equal time: every strategy's spp is calibrated so that its render takes
    # about as long as DARTS at the config's spp
    _, ms_d0, _ = _render(dts, torch, c, spp, 1)
    paths_px = spp * (c["n_bins"] if c["spp_mode"] == "cell" else 1)
    for strat in strategies:
        if strat == "vanilla":
            cs = dict(c, strategy="vanilla")
            s0 = paths_px
        elif strat == "uniform_s":
            cs = dict(c, conn_sampling="uniform")
            s0 = spp
        else:
            cs = dict(c, strategy=strat)
            s0 = spp
        if strat == "darts":
            sk = spp
        else:
            _, ms0, _ = _render(dts, torch, cs, s0, 2)
            sk = max(1, int(round(s0 * ms_d0 / max(ms0, 1e-3))))
        reps = []
        for r in range(nreps):
            h, ms, cnt = _render(dts, torch, cs, sk, 100 + r)
            reps.append({"ms": ms, "mse": float(((h - ref) ** 2).mean()), "vertices": cnt["vertices"]})
        ms = float(np.mean([x["ms"] for x in reps]))
        mse = float(np.mean([x["mse"] for x in reps]))
        med = float(np.median([x["mse"] for x in reps]))  # the stable statistic: the MSEs are heavy-tailed
        out["strategies"][strat] = {"spp": sk, "ms": ms, "mse": mse, "mse_median": med, "mse_x_ms": mse * ms,
                                    "mse_median_x_ms": med * ms, "reps": reps}
    base = out["strategies"]["darts"]["mse_x_ms"]
    base_med = out["strategies"]["darts"]["mse_median_x_ms"]
    for strat, v in out["strategies"].items():
        v["rel_mse_time_adjusted"] = v["mse_x_ms"] / base if base > 0 else None
        v["rel_median_mse_time_adjusted"] = v["mse_median_x_ms"] / base_med if base_med > 0 else None
    out["ref_signal_ms"] = float((ref ** 2).mean())
    print(f"cfg{idx}/{mode}: " + " | ".join(f"{k} spp {v['spp']} {v['ms']:.1f} ms MSE {v['mse']:.3e} "
                                          f"(x{v['rel_mse_time_adjusted']:.2f}, median x{v['rel_median_mse_time_adjusted']:.2f})"
                                          for k, v in out["strategies"].items()),
          flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--ref-mult", type=int, default=64)
    ap.add_argument("--strategies", nargs="+", default=["darts", "da_only", "eda_only", "uniform_s", "vanilla"],
                    help="darts first; MSE is reported relative to it at equal time (PAPER.md:433)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "mse_equal_time.json"))
    args = ap.parse_args()
    import torch

    from paper_2402_03106_b200 import dts
    res = []
    for idx in args.configs:
        modes = ["reuse", "split"] if idx in (3, 5) else [I.config(idx)["direction_mode"]]
        for m in modes:
            res.append(run_config(dts, torch, idx, m, args.reps, args.ref_mult, args.strategies))
            os.makedirs(os.path.dirname(args.out), exist_ok=True)
            with open(args.out, "w") as f:
                json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
