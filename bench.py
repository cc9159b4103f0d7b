#!/usr/bin/env python3
"""bench.py -- frames/sec of detect + 68 landmarks @640x480 on B200 (BASELINE.json metric).

Workload (one step, per GPU): B synthetic 640x480 eyeblink-camera frames (u8, seeded ring
targets) -> pyramid -> gradHist -> features -> tcgen05 fp16 screen -> exact fp64 re-score ->
threshold -> NMS -> ERT 15 x 500 x depth-4 random-init 68-landmark cascade on every kept
detection.  Models: the reference's own ring-pattern detector (tests/golden/
pattern_detector.npz, exported from the reference's pattern_detector()) and a seeded
random-init ERT.

Multi-GPU: frames are independent.  A step's global batch is
B x N frames of one global synthetic sequence; rank r owns the contiguous shard
sharding.shard_range(B*N, r, N) (B frames each: weak scaling, "scaling": "weak"), runs the
whole path on it with its own model replica, and the per-frame results are gathered on rank 0
in frame order after the timed region.  No collective on the data path; NCCL carries only the
barriers, the max-over-ranks timing reduction and the result gather.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B]     # our arm
  python bench.py --impl reference ...                                  # reference CPU arm

With --gpus N > 1 and no WORLD_SIZE in the environment, bench.py launches the N ranks itself
(RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR=127.0.0.1 / MASTER_PORT), one process per GPU;
under torchrun it uses the launcher's ranks.

`value` is device-resident throughput (frames already in HBM); `e2e` is the same metric
through the public C-ABI call with pinned host frames (H2D of the frames and D2H of all
detections + landmarks inside the timed region).  Each step's inputs (B*307 KB u8, 315 MB
at the default B=1024) exceed the 126 MB L2, so no explicit L2 flush is needed.  At N=1 the line also
carries `configs`: the other BASELINE.json configurations (C1 single-frame latency, C2, C3,
C5 throughput, C4 landmarks-only), each with its own e2e, roofline and CPU baseline.
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import os
import platform
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))

METRIC = "frames/sec detect+68 landmarks @640x480"
W, H = 640, 480
ERT_T, ERT_K, ERT_F = 15, 500, 4
# the other BASELINE.json configs measured at N=1 (name, w, h, frames per batch)
CONFIGS = (("C2", 320, 240, 16), ("C3", 1280, 720, 64), ("C5", 1920, 1080, 256))


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=40)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--batch", type=int, default=1024, help="frames per GPU per step")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-configs", action="store_true", help="skip the C1-C5 sub-measurements")
    p.add_argument("--launcher-selftest", action="store_true",
                   help="spawn/rendezvous check only (gloo, no GPU): rank 0 prints the ranks it saw")
    return p.parse_args()


def load_synthetic():
    """paper_2006_00816_b200/synthetic.py by file path: numpy only, so the reference arm never
    maps the GPU library (importing the package would)."""
    spec = importlib.util.spec_from_file_location("_bl_synthetic",
                                                  os.path.join(ROOT, "paper_2006_00816_b200", "synthetic.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def reference():
    """The reference CPU library (oracle/_ref) through its ctypes face -- the checker and the
    CPU baseline; never the thing measured for our arm."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference
    return Reference()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_models():
    syn = load_synthetic()
    g = np.load(os.path.join(ROOT, "tests", "golden", "pattern_detector.npz"))
    det = {"weights": np.tile(g["weights"], (5, 1)), "biases": np.full(5, float(g["bias"])),
           "threshold": float(g["threshold"])}
    ert = syn.random_ert(L=68, T=ERT_T, K=ERT_K, F=ERT_F, seed=2020)
    return det, ert


def frames_range(begin, end, w=W, h=H):
    """Frames [begin, end) of the global synthetic sequence: a 0.5*min(w,h) ring, centre
    jittered +-10% per frame (detected at pyramid level ~6 at 640x480)."""
    return load_synthetic().ring_frames_range(begin, end, w, h, seed=1000)


def tiled_frames(n, w, h, distinct=16, seed=77):
    """n frames cycling through `distinct` generated ones (large configs: generation time)."""
    syn = load_synthetic()
    base = syn.ring_frames_np(min(n, distinct), w, h, seed=seed)
    return np.ascontiguousarray(base[np.arange(n) % len(base)])


def host_cpu():
    """Cores this process may use (affinity) and the CPU model name."""
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        cores = os.cpu_count() or 1
    model = platform.processor() or "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return cores, model


# ------------------------------------------------------------------- launcher
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(a):
    """One process per GPU: RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* set here, as torchrun
    would (the driver may also launch bench.py under torchrun; then this is not used)."""
    n = a.gpus
    port = free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rcs = [p.wait() for p in procs]
    return max(rcs, key=abs) if any(rcs) else 0


def launcher_selftest(a):
    import torch.distributed as dist
    rank, world, local = dist_env()
    dist.init_process_group("gloo", init_method="env://")
    seen = [None] * world
    dist.all_gather_object(seen, {"rank": rank, "local_rank": local, "world": world, "pid": os.getpid()})
    if rank == 0:
        print(json.dumps({"launcher": "bench.py", "n_gpus": world, "ranks": seen}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------- roofline accounting
def geometry(w=W, h=H):
    """Pyramid geometry of a workload (image.cpp:158-172 + detector.cpp:144-167)."""
    lw, lh = [w], [h]
    while True:
        nw, nh = lw[-1] * 5 // 6, lh[-1] * 5 // 6
        if nw < 80 or nh < 80:
            break
        lw.append(nw)
        lh.append(nh)
    min_face = 0.2 * min(w, h)
    scored = [k for k in range(len(lw)) if 80 / (5 / 6) ** k >= min_face * (1 - 1e-9) and lw[k] // 8 >= 10
              and lh[k] // 8 >= 10]
    return lw, lh, scored


# fp64 operations per level pixel in the fused gradHist: gx, gy (2 sub), s = gx^2 + gy^2
# (2 mul + add), sqrt_fast (4 mul + 4 fma), then per neighbouring cell m*wx and (m*wx)*wy
# for two open cell rows plus the two adds (2 x 5)
GRADHIST_FP64_OPS = 2 + 3 + 8 + 10


def algorithmic_bytes_per_frame(w=W, h=H):
    """Canonical per-frame bytes of each stage."""
    lw, lh, scored = geometry(w, h)
    res = sum((1 if k == 1 else 8) * lw[k - 1] * lh[k - 1] + 8 * lw[k] * lh[k] for k in range(1, len(lw)))
    cells = sum((lw[k] // 8) * (lh[k] // 8) for k in scored)
    px = sum((1 if k == 0 else 8) * lw[k] * lh[k] for k in scored)
    anchors = sum((lw[k] // 8 - 9) * (lh[k] // 8 - 9) for k in scored)
    return {
        "pyramid": res,
        "gradhist": px + cells * 19 * 8,                  # level pixels read, bins + energy written
        "gradhist_px": sum(lw[k] * lh[k] for k in scored),  # level pixels (fp64 ops: GRADHIST_FP64_OPS each)
        "features": cells * (19 * 8 + 31 * 8 + 32 * 2),  # bins+energy read, fp64 + fp16 planes written
        "screen": cells * 32 * 2,                         # fp16 feature planes read once
        "anchors": anchors,
        "cells": cells,
    }


def ert_bytes_per_face():
    # touched per face: T*K leaf rows (L*2 doubles) + F split records (48 B) + 2F pixels
    return ERT_T * ERT_K * (68 * 2 * 8 + ERT_F * 48 + ERT_F * 2)


def load_peaks():
    peaks, note = {}, "fallback (B200_PROFILING.md: 6650 GB/s, 1590 bf16 TFLOP/s; MEASURED_PEAKS.json absent)"
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        note = "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    sec = {}
    try:  # secondary denominators measured on the box by tools/peaks.cu
        sec = json.load(open(os.path.join(ROOT, "profiles", "peaks_b200.json")))
    except Exception:
        pass
    return float(peaks.get("hbm_gbs", 6650.0)), float(peaks.get("bf16_tflops", 1590.0)), note, sec


def stage_table(stages, w, h, B, faces_per_step):
    """Per-stage ms, algorithmic GB/s and fraction of the bounding peak; the dominant kernel's
    roofline object."""
    hbm_peak, f16_peak, note, sec = load_peaks()
    alg = algorithmic_bytes_per_frame(w, h)
    traffic = {}
    if (w, h) == (W, H):
        try:  # ncu dram__bytes_read + write per frame of each stage's kernels (profiles/traffic.json)
            traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["bytes_per_frame"]
        except Exception:
            pass
    kern_ms = {k: stages.get(k, 0.0) for k in ("pyramid", "gradhist", "features", "screen", "rescore", "nms", "ert")}
    ert_bytes = faces_per_step * ert_bytes_per_face()
    bytes_stage = {"pyramid": alg["pyramid"] * B, "gradhist": alg["gradhist"] * B, "features": alg["features"] * B,
                   "screen": alg["screen"] * B, "ert": ert_bytes}
    per = {}
    for k, ms in kern_ms.items():
        e = {"ms": round(ms, 4)}
        if k in bytes_stage and ms > 0:
            gbs = bytes_stage[k] / (ms / 1000.0) / 1e9
            e.update({"GB/s": round(gbs, 1), "frac_hbm": round(gbs / hbm_peak, 3)})
        if k in traffic:
            e["dram_GB_ncu"] = round(traffic[k] * B / 1e9, 3)
        per[k] = e
    if sec and kern_ms["gradhist"] > 0:
        ops = GRADHIST_FP64_OPS * alg["gradhist_px"] * B / (kern_ms["gradhist"] / 1000.0) / 1e12
        per["gradhist"].update({"fp64_Tops": round(ops, 2), "frac_fp64": round(ops / sec["fp64_add_tflops"], 3)})
    if sec and kern_ms["ert"] > 0:
        per["ert"]["frac_l2"] = round(ert_bytes / (kern_ms["ert"] / 1000.0) / 1e9 / sec["l2_read_gbs"], 3)
    if kern_ms["screen"] > 0:  # the tcgen05 screen: useful FLOPs (dense 10x10x31 x 5 filters)
        tfs = 2 * 5 * 3100 * alg["anchors"] * B / (kern_ms["screen"] / 1000.0) / 1e12
        per["screen"].update({"TFLOP/s": round(tfs, 1), "frac_f16": round(tfs / f16_peak, 3)})
    # dominant HBM-bound kernel of the detection path (the ERT cascade is L1/L2-bound: its
    # "touched bytes" are reported in stages_ms.ert, not as an HBM roofline)
    dom = max((k for k in ("pyramid", "gradhist", "features", "screen")), key=lambda k: kern_ms[k])
    ach = bytes_stage[dom] / (kern_ms[dom] / 1000.0) / 1e9 if kern_ms[dom] > 0 else 0.0
    roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
            "frac": round(ach / hbm_peak, 3),
            "traffic": round(traffic[dom] * B / 1e9, 3) if dom in traffic else None,
            "traffic_unit": "GB per step (ncu dram__bytes_read+write.sum, profiles/traffic.json)",
            "peak_source": note, "kernel": dom,
            "bytes_per_step": int(bytes_stage[dom]),
            "bytes_per_frame_note": f"{dom}: {alg[dom]} algorithmic B/frame (DESIGN.md §5) x {B} frames"}
    return per, roof


# ------------------------------------------------------------------------ our arm
def pipelined(ctx, bl, src, k, landmarks=True):
    """k batches through the public submit/collect API (bl.MAX_IN_FLIGHT in flight: H2D,
    detection and the landmark cascade of different batches overlap).  Returns faces of the
    last batch."""
    faces = 0
    pending = [ctx.submit(src, landmarks=landmarks) for _ in range(min(k, bl.MAX_IN_FLIGHT))]
    issued = len(pending)
    while pending:
        res = ctx.collect(pending.pop(0), flat=True)
        faces = len(res[0])
        if issued < k:
            pending.append(ctx.submit(src, landmarks=landmarks))
            issued += 1
    return faces


def timed(torch, stream, fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    r = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1000.0, time.perf_counter() - t0, r


def stage_pass(ctx, bl, dev_frames, reps=3):
    ctx.enable_stage_timing(True)
    acc = {k: 0.0 for k in bl.STAGES}
    for _ in range(reps):
        ctx.detect_landmarks(dev_frames, flat=True)
        for k, v in ctx.stage_times().items():
            acc[k] += v / reps
    ctx.enable_stage_timing(False)
    return acc


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2006_00816_b200 as bl
    from paper_2006_00816_b200.sharding import max_over_ranks as _mor, run_sharded, shard_range

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL's own INFO log (ranks, transports) on stderr; stdout keeps the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device(f"cuda:{local}"))
    det, ert = load_models()
    B = args.batch
    G = B * world
    begin, end = shard_range(G, rank, world)
    frames = frames_range(begin, end)
    ctx = bl.Context(local)
    ctx.upload_detector(det)
    ctx.upload_ert(ert)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    dev_frames = torch.from_numpy(frames).cuda()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        return _mor(x, device=torch.device("cuda", local))

    # ---- device-resident timed region
    faces_per_step = pipelined(ctx, bl, dev_frames, max(3, args.warmup))
    barrier()
    l0 = ctx.launch_count
    with ClockSampler(local) as clk:
        t_dev_local, t_wall, _ = timed(torch, stream, lambda: pipelined(ctx, bl, dev_frames, args.steps))
    launches = ctx.launch_count - l0
    barrier()
    t_dev = max_over_ranks(t_dev_local)
    value = G * args.steps / t_dev

    stages = stage_pass(ctx, bl, dev_frames, max(1, min(3, args.steps)))

    # ---- end-to-end through the public call with pinned host frames
    e2e = None
    if not args.no_e2e:
        host = torch.from_numpy(frames).pin_memory().numpy()
        pipelined(ctx, bl, host, max(1, args.warmup))
        barrier()
        t_e, t_w, n_faces = timed(torch, stream, lambda: pipelined(ctx, bl, host, args.steps))
        t_e2e = max_over_ranks(max(t_e, t_w))
        d2h = B * 4 + 12 + n_faces * (32 + 68 * 2 * 8)
        e2e = {"value": round(G * args.steps / t_e2e, 1), "unit": "frames/s",
               "h2d_bytes_per_step": B * W * H, "d2h_bytes_per_step": d2h,
               "api": f"bl_submit/bl_collect ({bl.MAX_IN_FLIGHT} batches in flight), pinned host frames"}

    per_stage, roofline = stage_table(stages, W, H, B, faces_per_step)
    if roofline["kernel"] == "gradhist":
        roofline["limiter"] = ("instruction issue / fp64 pipe (ncu: profiles/, DESIGN.md §5): the exact fp64 "
                               "gradient, orientation and histogram per level pixel")

    # ---- shard -> run -> gather of the per-frame results (outside the timed region): rank 0
    # holds the global batch's detections per frame in frame order
    def per_frame(fr):
        dets, counts, _ = ctx.detect_landmarks(torch.from_numpy(fr).cuda(), flat=True)
        offs = np.concatenate([[0], np.cumsum(counts)])
        return [(int(counts[i]), float(np.sum(dets["score"][offs[i]:offs[i + 1]]))) for i in range(len(counts))]

    _, _, local_res, gathered = run_sharded(G, rank, world, lambda b, e: frames, per_frame)
    rank_info = {"rank": rank, "local_rank": local, "device": torch.cuda.get_device_name(local),
                 "pci_bus_id": torch.cuda.get_device_properties(local).pci_bus_id
                 if hasattr(torch.cuda.get_device_properties(local), "pci_bus_id") else None,
                 "shard": [begin, end], "device_s": round(t_dev_local, 5),
                 "faces": int(sum(c for c, _ in local_res))}
    ranks = [rank_info]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, rank_info)

    # ---- CPU baseline (rank 0, N=1): the reference library on this box's cores
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(frames, det, ert, n=64, budget_s=10.0)

    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        # a fresh context: the configs' own plans and pinned staging, not the bench batch's
        # (the main context's ~20 GB of lane arenas and slot buffers are released first)
        ctx.close()
        cctx = bl.Context(local)
        cctx.upload_detector(det)
        cctx.upload_ert(ert)
        cctx.set_stream(stream.cuda_stream)
        configs = measure_configs(args, torch, bl, cctx, stream, det, ert)
        cctx.close()

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_dev / args.steps * 1000.0, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(B, world, faces_per_step),
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk.summary(),
        "gpu_launches": int(launches), "stages_ms": per_stage,
        "ms_per_step_wall": round(t_wall / args.steps * 1000.0, 3),
        "ranks": ranks,
        "gathered": {"frames": len(gathered) if gathered is not None else None,
                     "faces": int(sum(c for c, _ in gathered)) if gathered is not None else None,
                     "how": "sharding.run_sharded: per-rank shard -> detect+landmarks -> gather_object in frame order"},
        "configs": configs,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def config_dict(B, world, faces_per_step=None):
    d = {"workload": f"{W}x{H} synthetic ring frames (u8), reference pattern detector (5 filters), "
                     f"ERT {ERT_T}x{ERT_K}xdepth{ERT_F} random-init 68 landmarks on every kept detection",
         "frames_per_gpu_per_step": B, "global_batch": B * world,
         "parallelism": f"frame shards (shard_range of the global batch), {world} independent replicas, "
                        "no data-path collective",
         "l2": f"inputs larger than L2 ({B * W * H / 1e6:.0f} MB u8 frames per GPU per step > 126 MB)"}
    if faces_per_step is not None:
        d["faces_per_step_per_gpu"] = faces_per_step
    return d


def measure_configs(args, torch, bl, ctx, stream, det, ert):
    """C1-C5 of BASELINE.json at N=1, each with device-resident value, e2e (pinned host frames
    through submit/collect), roofline of its dominant detection kernel and a bounded CPU
    baseline (the reference library on all host threads)."""
    ref = reference()
    cores, _ = host_cpu()
    out = {}
    for name, w, h, b in CONFIGS:
        # enough batches that the 4-deep pipeline's fill and drain (a batch's full latency at
        # each end) stay a small fraction of the timed region: ~0.1 s or 40 steps, whichever more
        steps = max(10, args.steps, int(0.8e9 / (b * w * h)))  # (~8 G px/s: 0.1 s)
        fr = tiled_frames(b, w, h)
        dev = torch.from_numpy(fr).cuda()
        faces = pipelined(ctx, bl, dev, 20)
        t, _, _ = timed(torch, stream, lambda: pipelined(ctx, bl, dev, steps))
        host = torch.from_numpy(fr).pin_memory().numpy()
        pipelined(ctx, bl, host, 20)
        te, tw, _ = timed(torch, stream, lambda: pipelined(ctx, bl, host, steps))
        st = stage_pass(ctx, bl, dev, 2)
        per, roof = stage_table(st, w, h, b, faces)
        cfps, nsample, dt = cpu_rate(ref, fr, det, ert, cores, budget_s=4.0)
        out[name] = {"workload": f"{w}x{h} x{b} frames per batch, detect + 68 landmarks",
                     "value": round(b * steps / t, 1), "unit": "frames/s", "ms_per_batch": round(t / steps * 1e3, 4),
                     "batches_timed": steps,
                     "faces_per_batch": faces,
                     "e2e": {"value": round(b * steps / max(te, tw), 1), "unit": "frames/s",
                             "h2d_bytes_per_step": b * w * h, "d2h_bytes_per_step": b * 4 + faces * (32 + 68 * 16)},
                     "roofline": roof, "stages_ms": per,
                     "cpu_baseline": {"value": round(cfps, 2), "unit": "frames/s", "cores": cores,
                                      "kind": "reference", "sample": f"{nsample} frames, {dt:.1f} s"}}
        del dev
    # C1: one 640x480 frame per batch, one batch in flight (latency), and 4 in flight
    fr = frames_range(0, 1)
    dev = torch.from_numpy(fr).cuda()
    host = torch.from_numpy(fr).pin_memory().numpy()
    pipelined(ctx, bl, dev, 20)
    n1 = 200

    def serial(src):
        for _ in range(n1):
            ctx.collect(ctx.submit(src), flat=True)
    t1, _, _ = timed(torch, stream, lambda: serial(dev))
    t1e, t1w, _ = timed(torch, stream, lambda: serial(host))
    t4, _, _ = timed(torch, stream, lambda: pipelined(ctx, bl, dev, n1))
    st = stage_pass(ctx, bl, dev, 5)
    per, roof = stage_table(st, W, H, 1, 3)
    single = cpu_single_thread(ref, fr, det, ert)
    out["C1"] = {"workload": "one 640x480 frame per batch, detect + 68 landmarks",
                 "latency_ms": round(t1 / n1 * 1e3, 4), "value": round(n1 / t1, 1), "unit": "frames/s",
                 "value_4_in_flight": round(n1 / t4, 1),
                 "e2e": {"value": round(n1 / max(t1e, t1w), 1), "unit": "frames/s",
                         "latency_ms": round(max(t1e, t1w) / n1 * 1e3, 4), "h2d_bytes_per_step": W * H,
                         "d2h_bytes_per_step": 4 + 3 * (32 + 68 * 16)},
                 "roofline": roof, "stages_ms": per,
                 "cpu_baseline": {"value": round(1000.0 / single["median_ms"], 3), "unit": "frames/s", "cores": 1,
                                  "kind": "reference", "sample": single["sample"],
                                  "median_ms_per_frame": single["median_ms"]}}
    out["C4"] = measure_c4(torch, bl, ctx, stream, ert, ref, cores)
    out["run"] = measure_run(bl, ctx, det, ert, ref, cores)
    return out


def measure_run(bl, ctx, det, ert, ref, cores, n=1024, n_ref=256, batch=64, repeats=3):
    """run() end to end (pipeline.cpp:396-404): a directory of n 640x480 PGM frames -> decode,
    detect, the best face's 68 landmarks, EAR trace.  Ours: bl_run (persistent decoder thread
    into pinned buffers, BL_MAX_IN_FLIGHT batches in flight) over n frames, the median of
    `repeats` timed runs (a 256-frame run is dominated by start-up: 1.3-2.7k frames/s against
    6-9.5k over 1024); reference: its pipelined run() with all usable host threads as workers
    over the first n_ref frames (a bounded sample; its rate is compute-bound and flat).  Wall
    clock, PGM decode included on both sides; the first n_ref frames' results are compared."""
    import shutil
    import tempfile
    d = tempfile.mkdtemp(prefix="bl_run_")
    dr = tempfile.mkdtemp(prefix="bl_run_ref_")
    try:
        for i, f in enumerate(tiled_frames(n, W, H, distinct=32, seed=91)):
            bl.write_pgm(os.path.join(d, f"frame_{i:06d}.pgm"), f)
            if i < n_ref:
                bl.write_pgm(os.path.join(dr, f"frame_{i:06d}.pgm"), f)
        ctx.run(d, 30.0, batch_size=batch)  # warm-up (plans, graphs, page cache)
        times = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            ours = ctx.run(d, 30.0, batch_size=batch)
            times.append(time.perf_counter() - t0)
        t_ours = float(np.median(times))
        ref.run(dr, det, ert, 30.0, pipelined=cores, batch_size=16)  # warm-up
        t0 = time.perf_counter()
        want = ref.run(dr, det, ert, 30.0, pipelined=cores, batch_size=16)
        t_ref = time.perf_counter() - t0
        nd = int(np.sum(ours["frames"]["n_detections"][:n_ref]))
        same = bool(np.array_equal(ours["detections"][:nd], want["detections"]) and
                    np.array_equal(ours["frames"]["face_found"][:n_ref], want["face_found"]))
    finally:
        shutil.rmtree(d, ignore_errors=True)
        shutil.rmtree(dr, ignore_errors=True)
    return {"workload": f"run(): {n} PGM frames {W}x{H}, decode + detect + best-face landmarks + EAR trace",
            "value": round(n / t_ours, 1), "unit": "frames/s", "batch_size": batch,
            "timing": f"median of {repeats} runs over {n} frames",
            "reference": {"value": round(n_ref / t_ref, 2), "unit": "frames/s", "workers": cores,
                          "kind": "reference run(), pipelined", "sample_frames": n_ref},
            "detections_identical": same}


def measure_c4(torch, bl, ctx, stream, ert, ref, cores):
    """C4: landmarks only, 10k random face boxes (side 120-279) in a 640x480 random-texture
    frame through the 15x500xdepth-4 cascade."""
    r = np.random.default_rng(405)
    n = 10000
    side = r.integers(120, 280, n)
    boxes = np.stack([r.integers(0, 640 - side + 1), r.integers(0, 480 - side + 1), side, side], 1).astype(np.int32)
    img = np.floor(np.random.default_rng(404).uniform(0, 256, (480, 640))).astype(np.uint8)
    ff = np.zeros(n, np.int32)
    ctx.landmarks(img, ff, boxes)  # warm-up
    d_img = torch.from_numpy(img[None]).cuda()
    d_ff = torch.from_numpy(ff).cuda()
    d_bx = torch.from_numpy(boxes).cuda()
    reps = 5
    t_dev, _, _ = timed(torch, stream, lambda: [ctx.landmarks(d_img, d_ff, d_bx) for _ in range(reps)])
    t_dev /= reps
    t_e2e, t_w, _ = timed(torch, stream, lambda: [ctx.landmarks(img, ff, boxes) for _ in range(reps)])
    t_e2e = max(t_e2e, t_w) / reps
    k = 2000
    ref.landmarks_batch_u8(img[None], ff[:cores], boxes[:cores], ert, cores)  # warm-up
    tc = time.perf_counter()
    ref.landmarks_batch_u8(img[None], ff[:k], boxes[:k], ert, cores)
    tcpu = time.perf_counter() - tc
    touched = ert_bytes_per_face() * n
    _, _, _, sec = load_peaks()
    l2 = float(sec.get("l2_read_gbs", 0)) or None
    ach = touched / t_dev / 1e9
    return {"workload": "10k boxes, landmarks only, 15x500xdepth4 ERT",
            "value": round(n / t_dev, 1), "unit": "boxes/s", "ms_per_10k": round(t_dev * 1e3, 3),
            "e2e": {"value": round(n / t_e2e, 1), "unit": "boxes/s", "h2d_bytes_per_step": 480 * 640 + n * 20,
                    "d2h_bytes_per_step": n * 68 * 16},
            "roofline": {"bound": "l2", "achieved": round(ach, 1), "peak": l2, "unit": "GB/s",
                         "frac": round(ach / l2, 3) if l2 else None, "kernel": "ert",
                         "note": "touched leaf+split+pixel bytes per face x faces / cascade time; peak = measured "
                                 "L2 read rate (profiles/peaks_b200.json)"},
            "cpu_baseline": {"value": round(k / tcpu, 1), "unit": "boxes/s", "cores": cores, "kind": "reference",
                             "sample": f"{k} boxes, {tcpu:.1f} s"}}


def cpu_rate(ref, frames, det, ert, threads, budget_s):
    ref.run_batch_u8(frames[:min(len(frames), threads)], det, ert, threads)  # warm-up
    n, t0, done = 0, time.perf_counter(), 0
    while time.perf_counter() - t0 < budget_s:
        chunk = np.roll(frames, -done, axis=0)[:threads] if len(frames) > threads else frames
        ref.run_batch_u8(chunk, det, ert, threads)
        n += len(chunk)
        done += len(chunk)
    dt = time.perf_counter() - t0
    return n / dt, n, dt


def cpu_single_thread(ref, frames, det, ert, reps=5):
    """Single-thread detect_faces + predict_landmarks per frame, median of `reps` after a
    discarded warm-up (pipeline.cpp:410-420's timing scheme)."""
    ref.run_batch_u8(frames[:1], det, ert, 1)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ref.run_batch_u8(frames[:1], det, ert, 1)
        ts.append((time.perf_counter() - t0) * 1e3)
    return {"median_ms": round(float(np.median(ts)), 3), "sample": f"{reps} runs of 1 frame on 1 thread (median)"}


def cpu_baseline(frames, det, ert, n, budget_s):
    """The UNMODIFIED reference (oracle/_ref) timed on this host: detect_faces + predict_landmarks
    on every kept detection, frame-parallel over all usable host threads (pipeline.cpp's
    scheme), plus the single-thread median."""
    try:
        ref = reference()
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "frames/s", "cores": 0, "kind": "unavailable", "sample": str(e)}
    threads, model = host_cpu()
    sample = np.ascontiguousarray(frames[:n])
    ref.run_batch_u8(sample[:threads], det, ert, threads)  # warm-up (page-in, model build)
    t0 = time.perf_counter()
    reps, faces = 0, 0
    while True:  # ~10-30 s of CPU work: repeat the sample until the budget is spent
        f, counts, _ = ref.run_batch_u8(sample, det, ert, threads)
        faces += f
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= budget_s or reps >= 200:
            break
    single = cpu_single_thread(ref, sample, det, ert)
    return {"value": round(n * reps / dt, 3), "unit": "frames/s", "cores": threads, "kind": "reference",
            "cpu_model": model,
            "sample": f"{n} distinct {W}x{H} frames x {reps} passes = {n * reps} frames, {faces} faces "
                      f"landmarked, {dt:.1f} s wall on {threads} threads",
            "single_thread": {"value": round(1000.0 / single["median_ms"], 3), "unit": "frames/s",
                              "median_ms_per_frame": single["median_ms"], "sample": single["sample"]}}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref: the unmodified /root/reference
    sources behind a thin extern "C" wrapper) on all usable host threads, same metric and
    workload; each step a bounded sample of the frames.  Never imports the GPU package."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    det, ert = load_models()
    threads, model = host_cpu()
    ref = reference()
    # sample per step: at least one frame per thread, at most the GPU arm's per-GPU batch,
    # sized so the K timed steps take about 60 s
    probe = frames_range(0, threads)
    t0 = time.perf_counter()
    ref.run_batch_u8(probe, det, ert, threads)  # warm-up + rate probe
    rate = threads / max(1e-3, time.perf_counter() - t0)
    n = int(min(args.batch, max(threads, rate * 60.0 / max(1, args.steps))))
    n = max(threads, (n // threads) * threads)
    frames = frames_range(0, n)
    for _ in range(max(0, min(args.warmup, 1))):
        ref.run_batch_u8(frames[:threads], det, ert, threads)
    t0 = time.perf_counter()
    faces = 0
    for _ in range(args.steps):
        f, _, _ = ref.run_batch_u8(frames, det, ert, threads)
        faces += f
    dt = time.perf_counter() - t0
    v = n * args.steps / dt
    cfg = config_dict(args.batch, world)
    cfg["reference_frames_per_step"] = n
    cfg["parallelism"] = f"frame-parallel std::threads x{threads} (host CPU, the reference's scheme)"
    line = {
        "metric": METRIC, "value": round(v, 3), "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1000, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": cfg,
        "cpu_baseline": {"value": round(v, 3), "unit": "frames/s", "cores": threads, "kind": "reference",
                         "cpu_model": model,
                         "sample": f"{n} frames per step x {args.steps} steps, {faces} faces landmarked"},
        "e2e": {"value": round(v, 3), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    import faulthandler
    faulthandler.enable()
    a = parse()
    sys.path.insert(0, ROOT)
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ and a.impl == "ours":
        sys.exit(spawn_ranks(a))
    if a.launcher_selftest:
        return launcher_selftest(a)
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    main()
