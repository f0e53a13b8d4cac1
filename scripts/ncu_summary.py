#!/usr/bin/env python
"""Summarise an ncu --set full capture of the render kernel (run HERE, no GPU):
pipe utilisation (fma / alu / xu), issue-slot use, SIMT efficiency, warp
stall reasons, atomics and DRAM traffic -> JSON (profiles/) + a text table.

    python scripts/ncu_summary.py gpurun_out/prof_c5.ncu-rep [--out profiles/ncu_r01_c5.json]
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.sum",
    "sm__inst_executed_pipe_alu.sum",
    "sm__inst_executed_pipe_xu.sum",
    "sm__inst_executed_pipe_lsu.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__shared_mem_per_block_dynamic",
    "launch__grid_size",
    "launch__block_size",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
    "lts__t_sectors_op_red.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smsp__average_warp_latency_issue_stalled_math_pipe_throttle",
]
STALL_PREFIX = "smsp__average_warps_issue_stalled_"


def read_raw(path: str) -> dict:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        raise SystemExit(f"no data in {path}")
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        recs.append({h: (v, u) for h, u, v in zip(hdr, units, r)})
    return recs


def summarise(rec: dict) -> dict:
    s = {"kernel": rec.get("Kernel Name", ("?", ""))[0]}
    for k in KEYS:
        if k in rec:
            s[k] = rec[k][0] + (f" {rec[k][1]}" if rec[k][1] else "")
    stalls = {}
    for k, (v, _u) in rec.items():
        if k.startswith(STALL_PREFIX) and k.endswith("_per_issue_active.ratio"):
            try:
                stalls[k[len(STALL_PREFIX):-len("_per_issue_active.ratio")]] = float(v.replace(",", ""))
            except ValueError:
                pass
    s["stalls_per_issue_active_top"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:10])
    return s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--out")
    a = ap.parse_args()
    recs = read_raw(a.rep)
    summ = [summarise(r) for r in recs]
    for s in summ:
        print(json.dumps(s, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(summ, f, indent=1)


if __name__ == "__main__":
    main()
