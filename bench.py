#!/usr/bin/env python
"""Benchmark: interlaced light-field frames/s of the CoherentRaster B200 path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One step = one interlaced frame through the whole hot path (SURVEY §8(a):
preprocess+SH with attribute reuse, tile/cluster binning, CUB-free radix sort,
ranges, remapped compositing) on synthetic scene_gen v1 data resident in HBM.
N>1 (torchrun, one process per GPU): the frame is split into row bands of
tiles, every rank renders its band, NCCL all-gathers the RGB8 bands; the
timed region is max over ranks (CUDA events, barrier + synchronize on both
sides).  Rank 0 prints ONE JSON line.  `--impl reference` times the CPU
oracle (the only reference this paper has) on a bounded band sample.
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

METRIC = "interlaced LF frames/s (4K, 100 views)"
METRICS = {"C": METRIC, "A": "interlaced LF frames/s (256x144, 8 views)",
           "B": "interlaced LF frames/s (4K, 45 views)", "D": "interlaced LF frames/s (8K, 100 views)",
           "E": "interlaced LF frames/s (4K, 45 views, 256 head-tracked poses)",
           "P2K": "interlaced LF frames/s (1440x2560 portrait, 63 views, s=16)",
           "P4K": "interlaced LF frames/s (4K, 71 views, s=18)"}
UNIT = "frames/s"
# algorithmic FP32 operations per (subpixel, splat) evaluation of Eqs.9-10,
# SURVEY §8d's count: delta 2, quadratic form 5, alpha
# (o exp, min) 3, transmittance 2, colour accumulation 2, tests 2 = 16,
# plus one MUFU exponential per evaluation.
FLOPS_PER_EVAL = 16
MUFU_PER_EVAL = 1


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def measure_traffic(cfg_name: str, s: int, kernel_regex: str = "k_composite_pairs|k_composite_staged"):
    """DRAM bytes (read + write) of one launch of the dominant kernel, from an
    ncu capture of one frame of the same config in a subprocess (after the
    timed region; ncu's replay never touches the timed numbers).  None when
    ncu is unavailable or not permitted on this box."""
    import csv
    import io
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control",
           "none", "-k", "regex:" + kernel_regex, "-c", "1", "--csv",
           sys.executable, os.path.join(ROOT, "tools", "prof_frame.py"), cfg_name, "1", str(s)]
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=240)
    except Exception:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tot, seen = 0.0, 0
    for row in csv.reader(io.StringIO(res.stdout)):
        if len(row) > 3 and row[-3] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            try:
                tot += float(row[-1].replace(",", "")) * scale.get(row[-2], 1.0)
                seen += 1
            except ValueError:
                pass
    return tot if seen == 2 else None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def compulsory_bytes(cfg, st):
    """SURVEY §8d B_c: scene + records + pairs + view map read + RGB8 write."""
    bg = 44 + 12 * (cfg.sh_degree + 1) ** 2
    S = cfg.W * cfg.H * 3
    return cfg.M * bg + 2 * st["visible_ik"] * 32 + st["pairs"] * (24 + 16 + 32) + 2 * S


def oracle_sample(cfg, scene, cams, rows, nthreads=0):
    """Time the CPU oracle (as it stands) on a band of tile rows of cfg."""
    import oracle
    o = oracle.Oracle(nthreads=nthreads)
    o.set_scene(scene)
    o.set_display(cfg.W, cfg.H, cfg.N, cfg.lens_pitch, slant=cfg.slant,
                  center_offset=cfg.center_offset)
    o.set_rig(cams)
    t0 = time.perf_counter()
    o.render(s=cfg.cluster_size, row0=rows[0], row1=rows[1])
    dt = time.perf_counter() - t0
    TY = (cfg.H + 15) // 16
    frac = (rows[1] - rows[0]) / TY
    return {"value": frac / dt, "unit": UNIT, "cores": o.threads, "kind": "oracle",
            "sample": (f"config {cfg.name} tile rows [{rows[0]},{rows[1]}) of {TY} "
                       f"({frac:.3f} of a frame: full preprocess of all {cfg.M} Gaussians x K "
                       f"clusters + band keys/sort/composite), {dt:.2f} s; frames/s = band "
                       "fraction / seconds (conservative: the per-frame preprocess is not "
                       "amortised over the band)"),
            "seconds": dt}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def workload(cfg) -> str:
    """The `config.workload` string both arms report for cfg."""
    return (f"config {cfg.name}: {cfg.M} Gaussians SH{cfg.sh_degree} "
            f"(scene_gen v1), {cfg.N}-view lenticular {cfg.W}x{cfg.H}")


def scaling_of(cfg) -> str:
    """Config E splits a fixed batch of poses per rank (weak); the others split one frame."""
    return "weak" if cfg.name == "E" else "strong"


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2605_04509_b200 import synthetic as sy  # noqa: F401
    scene, cams = cfg.make_scene(), cfg.make_rig()
    TY = (cfg.H + 15) // 16
    nr = max(1, min(args.ref_rows, TY))
    r0 = max(0, min(TY - nr, TY // 2 - nr // 2))
    rows = (r0, r0 + nr)
    for _ in range(args.warmup):
        oracle_sample(cfg, scene, cams, rows)
    times = []
    last = None
    for _ in range(args.steps):
        last = oracle_sample(cfg, scene, cams, rows)
        times.append(last["seconds"])
    frac = (rows[1] - rows[0]) / TY
    total = sum(times)
    value = args.steps * frac / total
    line = {
        "impl": "reference", "metric": METRICS.get(cfg.name, METRIC), "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / args.steps, "higher_is_better": True,
        "scaling": scaling_of(cfg), "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": workload(cfg), "cluster_size": cfg.cluster_size,
                   "parallelism": "CPU oracle on the host cores (band sample)",
                   "sample_tile_rows": list(rows)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": "oracle",
                         "sample": last["sample"], "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cluster-size", type=int, default=None)
    ap.add_argument("--no-remap", action="store_true")
    ap.add_argument("--kernel", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-traffic", action="store_true",
                    help="skip the ncu DRAM-traffic capture of the composite")
    ap.add_argument("--no-fullframe", action="store_true", help="skip the N1 full-frame comparator")
    ap.add_argument("--ref-rows", type=int, default=None,
                    help="oracle sample: tile rows (default 12 for cpu_baseline, 4 per --impl reference step)")
    ap.add_argument("--ablation", action="store_true", help="also time reuse/remap variants (stderr)")
    ap.add_argument("--refine", type=int, default=2,
                    help="band-split refinement rounds from measured band costs (N>1, balanced)")
    ap.add_argument("--bands", default="balanced", choices=["balanced", "equal"],
                    help="row-band split for N>1: equal-cost (calibration frame) or equal rows")
    args = ap.parse_args()

    from paper_2605_04509_b200 import synthetic as sy
    cfg = sy.CONFIGS[args.config]
    if args.cluster_size:
        cfg.cluster_size = args.cluster_size
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        if args.ref_rows is None:
            args.ref_rows = 4
        run_reference(args, cfg)
        return
    if args.ref_rows is None:
        args.ref_rows = 12

    import torch
    import torch.distributed as dist
    from paper_2605_04509_b200 import CoherentRaster

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # CR_BENCH_BACKEND=gloo (testing only): run N ranks on fewer GPUs through gloo
    backend = os.environ.get("CR_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    t_gen = time.perf_counter()
    scene, cams = cfg.make_scene(), cfg.make_rig()
    t_gen = time.perf_counter() - t_gen
    r = CoherentRaster(local)
    r.upload_gaussians(scene)
    r.set_display(cfg.W, cfg.H, cfg.N, cfg.lens_pitch, cfg.slant, cfg.center_offset, cfg.view_cone)
    r.set_camera_rig(cams)
    TX, TY = r.TX, r.TY
    from paper_2605_04509_b200.multigpu import BandGather, balanced_bands, row_pair_weights
    bands = None
    if world > 1 and args.bands == "balanced":
        # calibration frame (untimed): per-row pair counts -> equal-cost bands
        r.render(cfg.cluster_size)
        torch.cuda.synchronize()
        wrow = row_pair_weights(r, cfg.cluster_size) + 2.0e5
        bands = balanced_bands(wrow, world)
        # refine with MEASURED band costs (untimed): each rank renders its band,
        # the variable time (total minus the replicated preprocess) is gathered
        # and the per-row model rescaled band by band (multigpu.refine_bands)
        from paper_2605_04509_b200.multigpu import refine_bands
        cdev = dev if backend == "nccl" else torch.device("cpu")
        for _ in range(args.refine):
            cost = []
            for _ in range(3):
                r.render(cfg.cluster_size, rows=bands[rank], stats=True)
                st_ = r.last_stats
                cost.append(st_["ms_total"] - st_["ms_preprocess"])
            mine = torch.tensor([min(cost)], dtype=torch.float64, device=cdev)
            allc = torch.empty(world, dtype=torch.float64, device=cdev)
            dist.all_gather_into_tensor(allc, mine)
            bands, wrow = refine_bands(wrow, bands, allc.cpu().tolist(), world)
    bgt = BandGather(cfg.H, cfg.W, TY, world, rank, dev, bands=bands)
    rows = bgt.rows
    band_out = bgt.out
    remap = not args.no_remap
    kernel = args.kernel if args.kernel is not None else (0 if remap else 1)
    stream = torch.cuda.current_stream(dev)

    pose_mode = cfg.name == "E"
    if pose_mode:  # config E: head-tracked pose batch split round-robin over ranks
        from paper_2605_04509_b200.multigpu import pose_split
        poses = sy.head_tracked_poses(256, seed=1)
        my_poses = pose_split(len(poses), world, rank)
        pose_rigs = [cfg.make_rig(**poses[q]) for q in my_poses]
        rows = None
        band_out = torch.empty((cfg.H, cfg.W, 3), dtype=torch.uint8, device=dev)
        pose_i = [0]

    def step(stats=False, count=False):
        if pose_mode:
            r.set_camera_rig(pose_rigs[pose_i[0] % len(pose_rigs)])
            pose_i[0] += 1
            r.render(cfg.cluster_size, remap=remap, kernel=kernel, out=band_out, stats=stats,
                     count_evals=count)
            return
        r.render(cfg.cluster_size, remap=remap, kernel=kernel, rows=rows, out=band_out,
                 stats=stats, count_evals=count)
        bgt.gather()

    for _ in range(args.warmup):
        step()
    # one instrumented (untimed) frame: pairs, visible records, evaluation count
    step(stats=True, count=True)
    info = dict(r.last_stats)
    torch.cuda.synchronize()

    # ---- per-stage breakdown (untimed: stats synchronise after every frame)
    ms_stage = {"preprocess": 0.0, "bin": 0.0, "sort": 0.0, "composite": 0.0, "total": 0.0}
    nstage = min(5, args.steps)
    launches_per_step = 0
    for _ in range(nstage):
        step(stats=True)
        st = r.last_stats
        for k in ms_stage:
            ms_stage[k] += st["ms_" + k] / nstage
        launches_per_step = st["launches"]
    peak_ctx_bytes = int(r.last_stats["device_bytes"])

    # ---- timed region: back-to-back frames, a CUDA event after every step
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        evs[0].record(stream)
        for q in range(args.steps):
            step()
            evs[q + 1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [evs[q].elapsed_time(evs[q + 1]) for q in range(args.steps)]
    elapsed = evs[0].elapsed_time(evs[-1])  # ms
    t = torch.tensor([elapsed] + step_ms, dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t[0].item())
    step_ms = [float(v) for v in t[1:].tolist()]
    ms_per = elapsed / args.steps
    fps = args.steps / (elapsed / 1000.0)
    per_fps = sorted(1000.0 / max(v, 1e-9) for v in step_ms)
    pct = lambda p: per_fps[min(len(per_fps) - 1, int(round(p * (len(per_fps) - 1))))]  # noqa: E731
    mult = world if pose_mode else 1  # every rank renders its own pose frames
    fps *= mult
    fps_dist = {"p10": pct(0.10) * mult, "median": pct(0.5) * mult, "p90": pct(0.90) * mult,
                "unit": UNIT, "note": "per-step CUDA-event times (max over ranks per step)"}
    launches = launches_per_step * args.steps
    clocks = clk.summary()

    # ---- e2e: public API with host buffers (rig H2D + frame D2H every step).
    # At N=1 the frame goes to pinned host memory with async_out: the copy of
    # frame n overlaps the kernels of frame n+1 (two host buffers, two device
    # staging buffers inside the library); synchronize() inside the timed
    # region waits for the last copy, so every step's frame is on the host.
    hosts = [torch.empty((cfg.H, cfg.W, 3), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    host = hosts[0]
    rig_bytes = cams.astype(np.float32).nbytes
    e2e_i = [0]

    def e2e_step():
        r.set_camera_rig(cams)
        if pose_mode:
            step()
            host.copy_(band_out)
            return
        if world > 1:
            step()
            host.copy_(bgt.frame())
        else:
            e2e_i[0] ^= 1
            r.render(cfg.cluster_size, remap=remap, kernel=kernel, out=hosts[e2e_i[0]].numpy(),
                     async_out=True)

    for _ in range(2):
        e2e_step()
    r.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    r.synchronize()
    torch.cuda.synchronize()
    w1 = time.perf_counter() - w0
    tw = torch.tensor([w1], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tw, op=dist.ReduceOp.MAX)
    e2e_fps = args.steps / float(tw.item()) * (world if pose_mode else 1)

    # ---- N1 comparator: full-frame render of every view + interlace
    ff = None
    if world == 1 and not args.no_fullframe:
        if pose_mode:
            r.set_camera_rig(pose_rigs[0])

        def ff_ms_per_frame(view_batch, nff):
            mode = dict(cluster_size=1, fullframe=True, remap=True, kernel=0,
                        view_batch=view_batch)
            r.render(out=band_out, **mode)
            fe0, fe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            fe0.record(stream)
            for _ in range(nff):
                r.render(out=band_out, **mode)
            fe1.record(stream)
            torch.cuda.synchronize()
            return fe0.elapsed_time(fe1) / nff

        nff = 3
        ff_ms = ff_ms_per_frame(0, nff)
        by_batch = {}
        for vb in (36, 1):  # the paper's "3DGS (batch=36)" and plain per-view 3DGS
            if vb < cfg.N:
                ms_b = ff_ms_per_frame(vb, 2)
                by_batch[str(vb)] = {"ms_per_frame": ms_b, "value": 1000.0 / ms_b,
                                     "speedup_of_ours": ms_b / ms_per}
        ff = {"value": 1000.0 / ff_ms, "unit": UNIT, "ms_per_frame": ff_ms, "frames": nff,
              "speedup_of_ours": ff_ms / ms_per, "view_batch": cfg.N, "by_view_batch": by_batch,
              "note": "traditional baseline: every view rendered full frame (own attributes, "
                      "RGB per pixel) then interlaced by V; same kernels' binning/sort; all N "
                      "views in one pass, and B views per pass (B=36 as the paper's batched "
                      "3DGS, B=1 plain 3DGS)"}

    # ---- s = 4 beside the s = 8 headline: reuse is visibly lossy at s = 8 on
    # this synthetic scene (profiles/r02/reuse_quality_config*.md), so the
    # throughput of the next smaller cluster size is reported too (untimed loop)
    s4 = None
    if world == 1 and not pose_mode and cfg.cluster_size > 4:
        for _ in range(2):
            r.render(4, out=band_out)
        fe0, fe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        fe0.record(stream)
        n4 = 5
        for _ in range(n4):
            r.render(4, out=band_out)
        fe1.record(stream)
        torch.cuda.synchronize()
        s4 = {"cluster_size": 4, "value": 1000.0 * n4 / fe0.elapsed_time(fe1), "unit": UNIT,
              "frames": n4}

    # ---- ablation (stderr only)
    if args.ablation and rank == 0:
        for name, s_, rm, kn in [("ours s=8 staged", cfg.cluster_size, True, 0),
                                 ("paper-style thread/subpixel, remap", cfg.cluster_size, True, 1),
                                 ("w/o remap (thread, raster order)", cfg.cluster_size, False, 1),
                                 ("w/o reuse (s=1), staged", 1, True, 0)]:
            for _ in range(2):
                r.render(s_, remap=rm, kernel=kn, rows=rows, out=band_out, stats=True)
            tot = {"ms_total": 0.0, "ms_composite": 0.0}
            n = 5
            for _ in range(n):
                r.render(s_, remap=rm, kernel=kn, rows=rows, out=band_out, stats=True)
                for k in tot:
                    tot[k] += r.last_stats[k]
            print(f"[ablation] {name}: total {tot['ms_total']/n:.2f} ms composite "
                  f"{tot['ms_composite']/n:.2f} ms pairs {r.last_stats['pairs']}", file=sys.stderr)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks, peaks_src = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    comp_ms = ms_stage["composite"]
    evals = info["evals"]
    achieved_tflops = evals * FLOPS_PER_EVAL / (comp_ms * 1e-3) / 1e12 if comp_ms > 0 else None
    peak_tflops = 148 * 128 * 2 * sm_max * 1e6 / 1e12
    # MUFU: 16 SFU lanes per SM (4 per SMSP) -> 148 x 16 x clock exponentials/s
    mufu_peak = 148 * 16 * sm_max * 1e6 / 1e12
    mufu_ach = evals * MUFU_PER_EVAL / (comp_ms * 1e-3) / 1e12 if comp_ms > 0 else None
    bc = compulsory_bytes(cfg, info) if world == 1 else None
    # the composite's DRAM bytes per launch (ncu subprocess, after the timed region)
    traffic = (measure_traffic(args.config, cfg.cluster_size)
               if world == 1 and not args.no_traffic and not pose_mode else None)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rows_s = (TY // 2 - args.ref_rows // 2, TY // 2 - args.ref_rows // 2 + args.ref_rows)
        cpu = oracle_sample(cfg, scene, cams, rows_s)
        cpu.pop("seconds", None)
        cpu["cpu"] = cpu_model()
    line = {
        "metric": METRICS.get(cfg.name, METRIC), "value": fps, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per, "higher_is_better": True,
        "scaling": scaling_of(cfg), "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": workload(cfg),
                   "cluster_size": cfg.cluster_size, "remap": remap, "kernel": kernel,
                   "parallelism": (f"pose batch 256 split x{world}" if pose_mode else
                                   f"row-bands x{world} ({args.bands}: {bgt.bands or 'equal rows'})"
                                   if world > 1 else "single"),
                   "l2": "inputs larger than L2 (scene 0.7 GB, per-frame working set > 3 GB)",
                   "output": "RGB8 interlaced frame in HBM"},
        "pairs": info["pairs"], "visible_ik": info["visible_ik"], "evals": evals,
        "mean_traversal": evals / max(1, band_out.numel()),  # rank 0's band
        "stage_ms": ms_stage,
        "fps_distribution": fps_dist,
        "roofline": {"bound": "alu",
                     "kernel": ("k_composite_staged" if int(os.environ.get("CR_EXP", "0") or 0) & 64
                                else "k_composite_pairs"),
                     "achieved": achieved_tflops, "peak": peak_tflops, "unit": "TFLOP/s",
                     "frac": (achieved_tflops / peak_tflops) if achieved_tflops else None,
                     "traffic": traffic,
                     "mufu": {"achieved": mufu_ach, "peak": mufu_peak, "unit": "T exp/s",
                              "frac": (mufu_ach / mufu_peak) if mufu_ach else None},
                     "note": (f"{FLOPS_PER_EVAL} algorithmic FP32 ops + {MUFU_PER_EVAL} MUFU exp "
                              f"per (subpixel, splat) evaluation (SURVEY §8d) x {evals} "
                              "evaluations (the paper's traversal length, counted live by an "
                              "instrumented frame) / the composite's CUDA-event time in this "
                              f"run; peaks derived for {sm_max:.0f} MHz: 148 SM x 128 FP32 lanes "
                              "x 2 and 148 SM x 16 SFU lanes (DESIGN.md §5); traffic = DRAM "
                              "bytes read + written by one composite launch, ncu on one frame of "
                              "this config in a subprocess after the timed region (null: ncu "
                              "unavailable); algorithmic bytes per launch ~7.7 GB at C "
                              "(DESIGN.md §5)")},
        "frame_hbm": ({"compulsory_bytes": bc, "achieved_gbs": bc / (ms_per * 1e-3) / 1e9,
                       "peak_gbs": peaks.get("hbm_gbs"), "peak_source": peaks_src,
                       "frac": bc / (ms_per * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0)}
                      if bc else None),
        "clocks": clocks,
        "e2e": {"value": e2e_fps, "unit": UNIT, "h2d_bytes_per_step": int(rig_bytes),
                "d2h_bytes_per_step": int(cfg.W * cfg.H * 3),
                "note": "public API: cr_set_camera_rig from host + cr_render_interlaced into "
                        "pinned host memory (N=1: CR_FLAG_ASYNC_OUT, the D2H copy of frame n "
                        "overlapping frame n+1, cr_synchronize inside the timed region; wall "
                        "clock, max over ranks)"},
        "gpu_launches": launches,
        "memory": {"peak_context_device_bytes": peak_ctx_bytes,
                   "torch_max_allocated_bytes": int(torch.cuda.max_memory_allocated(dev)),
                   "note": "the library's device buffers (grow-only: the context's peak) + "
                           "torch's output / staging tensors"},
        "reuse_s4": s4,
        "cpu_baseline": cpu,
        "fullframe_baseline": ff,
        "scene_gen_s": t_gen,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
