"""Dump dts_sample_debug outputs for the parity records (analysis aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import dts_inputs as I
from paper_2402_03106_b200 import dts
os.makedirs("gpurun_out", exist_ok=True)
cases = [(1, "reuse"), (2, "reuse"), (3, "split"), (3, "reuse"), (4, "reuse"), (5, "split")]
if len(sys.argv) > 1:
    cases = [(int(a.split(":")[0]), a.split(":")[1]) for a in sys.argv[1:]]
for cfg, mode in cases:
    c = I.as_f32(I.config(cfg, direction_mode=mode))
    sc = dts.Scene(c); sc.table_build()
    recs = I.debug_records(c, 100_000, seed=100 + cfg)
    g = dts.debug(sc, recs)
    keep = ["tech", "p_hg", "p_eda", "p_mix", "ww", "wc", "t_lo", "t_hi", "hit", "conn_valid", "S", "t", "p_t",
            "contrib", "event", "cand_d", "cand_wn", "istar", "d", "beta_ris", "terminate", "S_lo", "S_hi", "p_m"]
    np.savez_compressed(f"gpurun_out/dbg_{cfg}_{mode}.npz", **{k: g[k] for k in keep})
print("ok")
