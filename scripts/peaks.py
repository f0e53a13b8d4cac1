#!/usr/bin/env python
"""Runs the pipe microbenchmarks of libdts_peaks.so (csrc/peaks.cu) on cuda:0
and prints/writes the per-SM-clock and per-second rates: the FP32 / MUFU /
issue denominators of the DARTS roofline.

    python scripts/peaks.py [--out gpurun_out/peaks.json]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = {0: "ffma_reg", 1: "ffma_imm", 2: "mufu_ex2", 3: "mufu_lg2", 4: "mufu_rsqrt", 5: "mufu_rcp", 6: "mufu_sin",
       7: "lop3", 8: "imad_wide+lop3", 9: "ffma+lop3", 10: "red_f32_global_random_4GB", 11: "red_f32_global_hot_4096",
       12: "atom_f32_shared"}


class Res(ctypes.Structure):
    _fields_ = [("ops", ctypes.c_double), ("ms", ctypes.c_double), ("mean_cycles", ctypes.c_double),
                ("grid", ctypes.c_int32), ("block", ctypes.c_int32)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "peaks.json"))
    ap.add_argument("--mhz", type=float, default=1965.0, help="SM clock the per-clock rates assume")
    args = ap.parse_args()
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2402_03106_b200", "libdts_peaks.so"))
    lib.dts_peak_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint32,
                                 ctypes.POINTER(Res)]
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = {"sms": sms, "gpu": torch.cuda.get_device_name(0), "ops": {}}
    try:
        out["nvidia_smi"] = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm",
                                            "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    except OSError:
        pass
    for op, name in OPS.items():
        iters = 16384 if op < 10 else 512
        r = Res()
        rc = lib.dts_peak_run(op, iters, 2, 1024, 1 << 30, ctypes.byref(r))
        if rc != 0:
            out["ops"][name] = {"error": rc}
            continue
        per_s = r.ops / (r.ms * 1e-3)
        # per SM clock at the max SM clock (the runs are seconds long at 1965 MHz, no throttling seen)
        per_clk_sm = per_s / (sms * args.mhz * 1e6)
        out["ops"][name] = {"thread_ops_per_s": per_s, "thread_ops_per_clk_per_sm_at_max_clock": per_clk_sm,
                            "fraction_of_issue_peak": per_s / (sms * 128 * args.mhz * 1e6), "ms": r.ms}
        print(f"{name:28s} {per_s:.3e} /s  {per_clk_sm:8.2f} thread-op/clk/SM at {args.mhz:.0f} MHz")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
