#!/usr/bin/env python
"""Benchmark of the DARTS hot path on B200 (BASELINE.json metric: path
vertices/s at 1/2/4/8 GPUs, as % of the FP32/SFU issue roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1)

One step = one complete render of the workload: zero the histogram, build the
EDA table (dts_table_build), render this rank's Philox sample range
(dts_render), and for N > 1 one NCCL reduce of the histograms to rank 0.
Strong scaling: the total work (config 5: 1024 spp per pixel) is split across
ranks by disjoint sample ranges.  Rank 0 prints ONE JSON line.

--impl reference times the fp64 CPU oracle (the only reference this paper
has) on a bounded sample of the same workload, on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import dts_inputs as I  # noqa: E402

# BASELINE.json's metric (the value is its first part: path vertices/s of the
# whole job; the roofline fraction is the JSON line's roofline.frac; the
# equal-time MSE is measured by scripts/mse_vs_oracle.py and mse_equal_time.py)
METRIC = "path vertices/s at 1/2/4/8 B200 (% FP32/SFU roofline); MSE vs oracle at equal time"
try:
    with open(os.path.join(ROOT, "BASELINE.json")) as _f:
        METRIC = json.load(_f).get("metric", METRIC)
except (OSError, ValueError):
    pass

# issue roofline: 148 SMs x 4 SMSPs x 32 lanes x 1 warp-instruction / clock
SMS, SMSP, LANES = 148, 4, 32
# the measured issue peak of the pipe microbenchmarks (FFMA + LOP3, 1965 MHz;
# profiles/peaks_r01.log): 3.662e13 thread-instructions/s
MEASURED_ISSUE_TIPS = 36.62


def _opcounts():
    with open(os.path.join(ROOT, "bench", "opcounts.json")) as f:
        return {k: v["ops"] for k, v in json.load(f)["vertex_types"].items()}


def algorithmic_instructions(counts: dict, mode: str) -> tuple[float, dict]:
    """Frozen algorithmic thread-instructions (bench/opcounts.json) summed over
    the measured vertex mix; returns (total, mix)."""
    ops = _opcounts()
    cam, wall, walk = counts["camera_vertices"], counts["wall_vertices"], counts["walk_vertices"]
    med = counts["vertices"] - cam - wall - walk
    mix = {"camera": cam, "wall": wall, "medium_split_walk_only": walk, f"medium_{mode}": med}
    return sum(n * ops[k] for k, n in mix.items()), mix


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _shard(spp: int, rank: int, world: int):
    from paper_2402_03106_b200.shard import shard_range
    return shard_range(spp, rank, world)


# --------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2402_03106_b200 import dts

    world, rank, local = _dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # communicator lines (rank count, NVLS / channels) for the driver, on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = I.as_f32(I.config(args.config, **({"ico_subdiv": args.mesh_subdiv} if args.config == 6 and
                                          args.mesh_subdiv is not None else {})))
    if args.direction_mode:
        c["direction_mode"] = args.direction_mode
    if args.strategy:
        c["strategy"] = args.strategy
    if args.spp:
        c["spp"] = args.spp
    if args.crop:
        c = I.crop_center(c, min(args.crop, c["width"]), min(args.crop, c["height"]))
    spp = c["spp"]
    sb, se = _shard(spp, rank, world)
    sc = dts.Scene(c)
    shape = sc.hist_shape()
    hist = torch.zeros(shape, dtype=torch.float32, device="cuda")
    ctr = torch.zeros(dts.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()

    kern_ms = []

    from paper_2402_03106_b200.shard import render_sharded, render_sharded_p2p

    def step(i, timed):
        sc.table_build(stream=stream)

        def render_range(b, e, target=None):  # this rank's disjoint Philox key range
            assert (b, e) == (sb, se)
            if timed:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            sc.render(spp, c["seed"] + 1000 * i, b, e, hist if target is None else target, None,
                      ctr if timed else None, stream)
            if timed:
                e1.record(stream)
                kern_ms.append((e0, e1))

        if args.reduce == "p2p":
            # fused: every rank's kernel adds straight into rank 0's histogram (peer memory)
            render_sharded_p2p(render_range, spp, hist, enable_peer=dts.enable_peer)
        else:
            # render the shard, then ONE reduce of the histograms to rank 0 (NCCL over NVLink)
            hist.zero_()
            render_sharded(render_range, spp, hist)

    for i in range(args.warmup):
        step(i, False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctr.zero_()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for i in range(args.steps):
            step(args.warmup + i, True)
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    kms = [a.elapsed_time(b) for a, b in kern_ms]
    kern_avg = sum(kms) / len(kms)
    launch = dts.last_launch()
    # per-rank step and render times (the rest of a step is the table build and,
    # at N > 1, the reduce); max over ranks of the step time; counters summed
    per_rank = {"step_ms": [ms / args.steps], "render_ms": [kern_avg]}
    if world > 1:
        mine = torch.tensor([ms / args.steps, kern_avg], dtype=torch.float64, device="cuda")
        allr = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        per_rank = {"step_ms": [float(t[0]) for t in allr], "render_ms": [float(t[1]) for t in allr]}
        tt = torch.tensor([ms, kern_avg], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, kern_avg = float(tt[0]), float(tt[1])
        dist.all_reduce(ctr, op=dist.ReduceOp.SUM)
    counts = dts.counters_dict(ctr)
    verts_per_step = counts["vertices"] / args.steps
    paths_per_step = counts["paths"] / args.steps

    # ---- end to end through the C ABI with HOST buffers (pinned), N GPUs
    e2e = None if args.no_e2e else run_e2e(args, c, sc, world, rank, stream, torch, dist, dts, ms / args.steps)

    if rank == 0:
        peaks = _peaks()
        sm_max = peaks.get("sm_max_mhz", 1965.0)
        mode = c["direction_mode"]
        alg_total, mix = algorithmic_instructions(counts, mode)
        alg = alg_total / max(counts["vertices"], 1)              # per vertex, over the measured mix
        peak_tips = SMS * SMSP * LANES * sm_max * 1e6 / 1e12      # Tinst/s at the max SM clock
        # the dominant kernel(s): the render's launches (two-stage: walk + connect),
        # per-rank algorithmic instructions / their CUDA-event time on the stream
        achieved = (verts_per_step / world) * alg / (kern_avg * 1e-3) / 1e12
        value = verts_per_step / (ms / args.steps * 1e-3)
        traffic = None if (args.spp or args.crop or args.strategy or args.direction_mode) else _profile_traffic(args.config)
        clocks = clk.summary()
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "vertices/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded Philox paths; analytic scene of BASELINE.json config)",
            "config": {
                "workload": c["name"], "config_index": args.config, "pixels": c["width"] * c["height"],
                "bins": c["n_bins"], "spp": spp, "spp_mode": c["spp_mode"], "direction_mode": mode,
                "paths_per_step": paths_per_step, "vertices_per_step": verts_per_step,
                **({"triangles": len(c["mesh"]["tris"])} if c.get("mesh") else {}),
                "parallelism": f"sample-range shards x{world}" + (
                    (" + fused peer-memory REDs" if args.reduce == "p2p" else " + NCCL reduce") if world > 1 else ""),
                "l2": ("histogram (%.2f GB) > L2 is re-zeroed every step" if hist.numel() * 4 > 126e6 else
                       "histogram (%.4f GB) fits L2 (small config: a parity case, not the headline); re-zeroed every step")
                      % (hist.numel() * 4 / 1e9),
            },
            "paths_per_s": paths_per_step / (ms / args.steps * 1e-3),
            "roofline": {
                "bound": "alu", "achieved": achieved, "peak": peak_tips, "unit": "Tinst/s",
                "frac": achieved / peak_tips, "frac_measured_peak": achieved / MEASURED_ISSUE_TIPS,
                # the frozen basis counts two Philox blocks at every vertex; a walk-only SPLIT
                # vertex draws one since the R24 re-layout: frac on that count
                "frac_walk_one_philox": achieved / peak_tips * (
                    1.0 - 51.5 * mix.get("medium_split_walk_only", 0) / max(alg * counts["vertices"], 1.0)),
                "traffic": traffic,
                "basis": f"{alg:.1f} algorithmic thread-instructions per vertex: bench/opcounts.json frozen counts "
                         f"x the measured vertex mix {{{', '.join(f'{k}: {v / max(counts['vertices'], 1):.4f}' for k, v in mix.items())}}}"
                         f" x vertices / render time (CUDA events); peak = 148 SM x 4 issue x 32 lanes x {sm_max:.0f} MHz "
                         f"(nominal); frac_measured_peak against the FFMA+LOP3 microbenchmark's {MEASURED_ISSUE_TIPS} Tinst/s"
                         + ("; BVH traversal of the mesh not counted" if c.get("mesh") else ""),
                "alg_instr_per_vertex": alg,
                "kernel_ms": kern_avg,
                "launches_per_step": launch.get("n_launches"),
            },
            "clocks": clocks,
            "per_rank": per_rank,
            "e2e": e2e,
            # per step and rank: the table build (2 kernels) + the render's launches
            # (two-stage: 2 per chunk; + 1 counter kernel when camera rays are culled)
            "gpu_launches": (2 + launch.get("n_launches", 1)) * args.steps * world,
            "launch": launch,
            "counters": counts,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_budget)
            if not args.no_mse:
                # the metric's second half, measured in this run
                line["mse_vs_oracle_equal_time"] = mse_equal_time(args.config, args.mse_seeds, args.mse_crop)
        print(json.dumps(line), flush=True)
    if world > 1:
        from paper_2402_03106_b200.shard import release_peer_histograms
        release_peer_histograms()
        torch.cuda.synchronize()
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, c, sc, world, rank, stream, torch, dist, dts, step_ms=1e9):
    from paper_2402_03106_b200.shard import pipeline_bands
    """Same metric through the public API with host buffers: per step the host
    scene description goes in (dts_scene_create + dts_table_build), the
    histogram comes back to pinned host memory."""
    cells = sc.hist_cells()
    # only rank 0 receives the histogram: only it pins a host buffer (4.2 GB for config 5)
    host = torch.empty(cells, dtype=torch.float32, pin_memory=True) if rank == 0 else None
    hnp = host.numpy() if host is not None else None
    hctr = np.zeros(dts.NUM_COUNTERS, np.uint64)
    spp = c["spp"]
    sb, se = _shard(spp, rank, world)
    # N > 1 (and DTS_E2E_BANDED=1 at N = 1, for testing): large histograms go band
    # by band -- render rows (dts_render_rows), reduce the band, and copy it to the
    # host on a copy stream while the next band renders
    banded_mode = world > 1 or os.environ.get("DTS_E2E_BANDED") == "1"
    dev_hist = torch.zeros(sc.hist_shape(), dtype=torch.float32, device="cuda") if banded_mode else None
    rows = c["crop"][3] - c["crop"][1]
    rowsz = (c["crop"][2] - c["crop"][0]) * c["n_bins"]
    nbands = 4 if (cells * 4 >= (256 << 20) and rows >= 8) else 1
    copy_stream = torch.cuda.Stream() if banded_mode else None
    verts = 0
    # at least 2 steps and ~0.5 s of work: millisecond configs are otherwise
    # dominated by the noise of a couple of host-side calls
    ksteps = max(1, min(args.steps, 2))
    if step_ms < 100.0:
        ksteps = max(ksteps, min(50, int(500.0 / max(step_ms, 1.0))))
    if world > 1:  # every rank must run the same number of collectives
        kt = torch.tensor([ksteps], dtype=torch.int64, device="cuda")
        dist.all_reduce(kt, op=dist.ReduceOp.MAX)
        ksteps = int(kt[0])
    for i in range(ksteps + 1):
        timed = i > 0
        if timed and i == 1:
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
        s2 = dts.Scene(c)
        s2.table_build(stream=stream)
        if not banded_mode:
            s2.render_host(spp, c["seed"] + 7 * i, sb, se, hnp, hctr, stream)
            if timed:
                verts += int(hctr[2])
        else:
            dev_hist.zero_()
            ctr = torch.zeros(dts.NUM_COUNTERS, dtype=torch.int64, device="cuda")
            flat = dev_hist.view(-1)

            def render_band(k, r0, r1, i=i, s2=s2, ctr=ctr):
                s2.render_rows(spp, c["seed"] + 7 * i, sb, se, r0, r1, k % 4, flat[r0 * rowsz:r1 * rowsz], ctr, stream)

            def reduce_band(k, r0, r1):
                # every collective stays on the main stream, in the same order on every rank
                dist.reduce(flat[r0 * rowsz:r1 * rowsz], dst=0)

            def copy_band(k, r0, r1):
                ev = torch.cuda.Event()
                ev.record(stream)
                copy_stream.wait_event(ev)
                with torch.cuda.stream(copy_stream):
                    host[r0 * rowsz:r1 * rowsz].copy_(flat[r0 * rowsz:r1 * rowsz], non_blocking=True)

            pipeline_bands(rows, nbands, render_band, reduce_band, copy_band, world, rank)
            if world > 1:
                dist.all_reduce(ctr)
            torch.cuda.synchronize()
            if timed:
                verts += int(ctr[2].item())
        s2.close()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([el], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = float(tt[0])
    import ctypes
    return {"value": verts / el, "unit": "vertices/s", "steps": ksteps,
            "h2d_bytes_per_step": ctypes.sizeof(dts.SceneDesc),
            "d2h_bytes_per_step": cells * 4 + (8 * dts.NUM_COUNTERS if world == 1 else 0),
            "timing": "host wall clock (perf_counter) around scene_create..histogram in pinned host memory, max over ranks"}


def _profile_traffic(cfg):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(str(cfg))
    except (OSError, ValueError):
        return None


# --------------------------------------------------------------------------- CPU oracle (cpu_baseline / reference arm)
def _oracle_sample(cfg_idx, crop_w, crop_h):
    from oracle import oracle as O
    c = I.as_f32(I.config(cfg_idx))
    c = I.crop_center(c, crop_w, crop_h)
    q = O.build_table(c)[0] if c["strategy"] == "darts" else None
    t = time.perf_counter()
    r = O.render(c, q, c["spp"], c["seed"], sq=False, nthreads=os.cpu_count())
    el = time.perf_counter() - t
    return r["stats"], el, c


def cpu_baseline(cfg_idx, budget_s=15.0):
    """The oracle as it stands on the host cores, on a bounded crop of the
    same workload (every bin and sample of the crop's pixels)."""
    w = 2
    st, el, c = _oracle_sample(cfg_idx, w, w)
    # grow the crop until the sample costs about budget_s
    while el < budget_s / 2 and w < 256:
        w2 = min(256, int(w * max(1.5, min(4.0, math.sqrt(budget_s / max(el, 1e-3) / 1.5)))))
        if w2 * w2 * (el / (w * w)) > 2.5 * budget_s:
            break
        w = w2
        st, el, c = _oracle_sample(cfg_idx, w, w)
    return {"value": st["vertices"] / el, "unit": "vertices/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"{c['name']} centre crop {w}x{w} px, all {c['n_bins']} bins, spp {c['spp']} "
                      f"({st['paths']} paths, {st['vertices']} vertices) in {el:.1f} s, fp64",
            "paths_per_s": st["paths"] / el}


def mse_equal_time(cfg_idx, seeds=16, crop=8):
    """BASELINE.json metric, second half: "MSE vs oracle at equal time"
    (the paper's equal-time MSE methodology).
    On a centre crop of the config (every bin, per-pixel spp as configured):
      1. the fp64 oracle renders the crop at the config's spp with ``seeds``
         seeds on all host cores; T_cpu = the median wall time of one render;
      2. the GPU renders the same crop at the sample count spp_eq it finishes
         in T_cpu (from a timed probe launch, refined once at the estimated
         count), DIRECTLY, with ``seeds`` seeds;
         each launch is timed (CUDA events) to show it took ~T_cpu;
      3. the reference for GPU seed k is the mean of the other seeds' renders
         (leave-one-out: (seeds - 1) x spp_eq samples, independent of render k);
         the oracle's reference is the mean of all GPU renders (seeds x spp_eq,
         thousands of times the oracle's count).  MSE over all crop cells.
    The reference's own error adds MSE_gpu / (seeds - 1) to each GPU MSE (reported,
    and removed in the corrected figure).  Per-path contributions are heavy-tailed
    (SURVEY 8(c.6)): the mean over seeds is dominated by rare paths, so the median
    is reported beside it.  An equal-spp GPU render (the oracle's count, same
    seeds protocol) checks that both estimators have the same MSE per sample."""
    import torch

    from oracle import oracle as O
    from paper_2402_03106_b200 import dts
    c0 = I.as_f32(I.config(cfg_idx))
    crop = min(crop, c0["width"], c0["height"])
    c = I.crop_center(c0, crop, crop)
    spp = c["spp"]
    q = O.build_table(c)[0]
    h_o, t_o = [], []
    for k in range(seeds):
        t = time.perf_counter()
        h_o.append(O.render(c, q, spp, 500 + k, sq=False, nthreads=os.cpu_count())["hist"])
        t_o.append(time.perf_counter() - t)
    t_cpu = statistics.median(t_o)
    sc = dts.Scene(c)
    sc.table_build()

    def gpu(n, seed):
        h = torch.zeros(sc.hist_shape(), dtype=torch.float32, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        sc.render(n, seed, 0, n, h)
        e1.record()
        torch.cuda.synchronize()
        return h.double().cpu().numpy(), e0.elapsed_time(e1) * 1e-3

    gpu(spp, 1)                                        # warm-up
    probe = 64 * spp
    _, t_probe = gpu(probe, 2)
    spp_eq = max(spp, int(probe * t_cpu / t_probe))
    _, t_1 = gpu(spp_eq, 3)                             # one refinement at the estimated count
    spp_eq = max(spp, int(spp_eq * t_cpu / t_1))
    h_g, t_g = [], []
    for k in range(seeds):
        h, t = gpu(spp_eq, 9000 + k)
        h_g.append(h)
        t_g.append(t)
    tot = np.sum(h_g, axis=0)
    mse_g_raw = [float(((h - (tot - h) / (seeds - 1)) ** 2).mean()) for h in h_g]
    mse_g = [m * (seeds - 1) / seeds for m in mse_g_raw]   # minus the leave-one-out reference's variance
    ref = tot / seeds
    mse_o = [float(((h - ref) ** 2).mean()) for h in h_o]
    h_s = [gpu(spp, 7000 + k)[0] for k in range(seeds)]
    mse_s = [float(((h - ref) ** 2).mean()) for h in h_s]
    med = statistics.median
    sc.close()
    return {
        "ratio_cpu_over_gpu_mean": float(np.mean(mse_o) / np.mean(mse_g)),
        "ratio_cpu_over_gpu_median": float(med(mse_o) / med(mse_g)),
        "mse_cpu": {"mean": float(np.mean(mse_o)), "median": med(mse_o)},
        "mse_gpu_equal_time": {"mean": float(np.mean(mse_g)), "median": med(mse_g),
                               "mean_uncorrected": float(np.mean(mse_g_raw))},
        "mse_gpu_equal_spp": {"mean": float(np.mean(mse_s)), "median": med(mse_s)},
        "t_cpu_s": t_cpu, "cpu_cores": os.cpu_count(), "spp_cpu": spp, "spp_gpu_equal_time": spp_eq,
        "t_gpu_s_median": med(t_g), "seeds": seeds,
        "crop": f"{c['name']} centre {crop}x{crop} px x {c['n_bins']} bins",
        "reference": f"GPU renders, leave-one-out mean of {seeds - 1} x spp_eq (GPU MSE), mean of {seeds} x spp_eq "
                     "(oracle MSE)",
    }


def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    for _ in range(args.warmup):
        _oracle_sample(args.config, 2, 2)
    tot_v, tot_t, last = 0, 0.0, None
    w = 4
    for _ in range(args.steps):
        st, el, c = _oracle_sample(args.config, w, w)
        tot_v += st["vertices"]
        tot_t += el
        last = (st, el, c)
    value = tot_v / tot_t
    st, el, c = last
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "vertices/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_t / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": c["name"], "config_index": args.config, "sample": f"centre crop {w}x{w}"},
        "cpu_baseline": {"value": value, "unit": "vertices/s", "cores": os.cpu_count(), "kind": "oracle",
                         "sample": f"{c['name']} centre crop {w}x{w} px x all bins x spp {c['spp']} per step"},
        "e2e": {"value": value, "unit": "vertices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5, 6])
    ap.add_argument("--direction-mode", choices=["reuse", "split"], default=None)
    ap.add_argument("--mesh-subdiv", type=int, default=None,
                    help="config 6: icosphere subdivision level (2 = 320 triangles, 6 = 81920)")
    ap.add_argument("--strategy", choices=["darts", "vanilla", "da_only", "eda_only"], default=None,
                    help="estimator (default: the config's, DARTS); other values are comparison runs, not bench lines")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--reduce", choices=["nccl", "p2p"], default="nccl",
                    help="N > 1: one NCCL reduce after the renders (default), or p2p: every rank's render "
                         "kernel adds into rank 0's histogram through CUDA IPC peer memory (no reduce)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg (A/B and profiling runs only)")
    ap.add_argument("--no-mse", action="store_true", help="skip the equal-time MSE against the oracle")
    ap.add_argument("--mse-seeds", type=int, default=16)
    ap.add_argument("--mse-crop", type=int, default=8)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--spp", type=int, default=None, help="override spp (profiling runs only; not a bench line)")
    ap.add_argument("--crop", type=int, default=None, help="centre crop W x W (profiling runs only; not a bench line)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
