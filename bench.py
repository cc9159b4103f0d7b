#!/usr/bin/env python3
"""bench.py -- frames/sec of detect + 68 landmarks @640x480 on B200 (BASELINE.json metric).

Workload (one step, per GPU): B synthetic 640x480 eyeblink-camera frames (u8, seeded ring
targets) -> pyramid -> gradHist -> features -> tcgen05 fp16 screen -> exact fp64 re-score ->
threshold -> NMS -> ERT 15 x 500 x depth-4 random-init 68-landmark cascade on every kept
detection.  Models: the reference's own ring-pattern detector (tests/golden/
pattern_detector.npz, exported from the reference's pattern_detector()) and a seeded
random-init ERT.  Frames are independent: N GPUs = N replicas with per-rank frame shards,
no collective on the data path ("scaling": "weak").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B]     # our arm
  python bench.py --impl reference ...                                  # reference CPU arm

`value` is device-resident throughput (frames already in HBM); `e2e` is the same metric
through the public C-ABI call with pinned host frames (H2D of the frames and D2H of all
detections + landmarks inside the timed region).  Each step's inputs (B*307 KB u8, 157 MB
at B=512) exceed the 126 MB L2, so no explicit L2 flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec detect+68 landmarks @640x480"
W, H = 640, 480
ERT_T, ERT_K, ERT_F = 15, 500, 4


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=40)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--batch", type=int, default=512, help="frames per GPU per step")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--ref-frames", type=int, default=32, help="reference arm: frames per step")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_models():
    from paper_2006_00816_b200.synthetic import random_ert
    g = np.load(os.path.join(ROOT, "tests", "golden", "pattern_detector.npz"))
    det = {"weights": np.tile(g["weights"], (5, 1)), "biases": np.full(5, float(g["bias"])),
           "threshold": float(g["threshold"])}
    ert = random_ert(L=68, T=ERT_T, K=ERT_K, F=ERT_F, seed=2020)
    return det, ert


def frames_for(rank, n):
    from paper_2006_00816_b200.synthetic import ring_frames_np
    # size 0.5*min(w,h) = 240 px ring, centre jittered +-10%: detected at pyramid level ~6
    return ring_frames_np(n, W, H, seed=1000 + rank)


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
def geometry():
    """Pyramid geometry of the workload (image.cpp:158-172 + detector.cpp:144-167)."""
    lw, lh = [W], [H]
    while True:
        nw, nh = lw[-1] * 5 // 6, lh[-1] * 5 // 6
        if nw < 80 or nh < 80:
            break
        lw.append(nw)
        lh.append(nh)
    min_face = 0.2 * min(W, H)
    scored = [k for k in range(len(lw)) if 80 / (5 / 6) ** k >= min_face * (1 - 1e-9) and lw[k] // 8 >= 10
              and lh[k] // 8 >= 10]
    return lw, lh, scored


# fp64 operations per level pixel in the fused gradHist: gx, gy (2 sub), s = gx^2 + gy^2
# (2 mul + add), sqrt_fast (4 mul + 4 fma), then per neighbouring cell m*wx and (m*wx)*wy
# for two open cell rows plus the two adds (2 x 5)
GRADHIST_FP64_OPS = 2 + 3 + 8 + 10


def algorithmic_bytes_per_frame():
    """Canonical per-frame bytes of each stage."""
    lw, lh, scored = geometry()
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


# ------------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2006_00816_b200 as bl

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device(f"cuda:{local}"))
    det, ert = load_models()
    B = args.batch
    frames = frames_for(rank, B)
    ctx = bl.Context(local)
    ctx.upload_detector(det)
    ctx.upload_ert(ert)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    dev_frames = torch.from_numpy(frames).cuda()

    def barrier():
        if world > 1:
            dist.barrier()

    from paper_2006_00816_b200.sharding import max_over_ranks as _mor

    def max_over_ranks(x):
        return _mor(x, device=torch.device("cuda", local))

    def run_steps(src, k):
        """k pipelined steps through the public submit/collect API (bl.MAX_IN_FLIGHT batches
        in flight: H2D, detection and the landmark cascade of different batches overlap)."""
        faces = 0
        pending = [ctx.submit(src) for _ in range(min(k, bl.MAX_IN_FLIGHT))]
        issued = len(pending)
        while pending:
            dets, counts, lms = ctx.collect(pending.pop(0), flat=True)
            faces = len(dets)
            if issued < k:
                pending.append(ctx.submit(src))
                issued += 1
        return faces

    # ---- device-resident timed region
    faces_per_step = run_steps(dev_frames, args.warmup)
    barrier()
    torch.cuda.synchronize()
    l0 = ctx.launch_count
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        tw0 = time.perf_counter()
        ev0.record(stream)
        run_steps(dev_frames, args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - tw0
    launches = (ctx.launch_count - l0) // max(1, args.steps)
    barrier()
    t_dev = max_over_ranks(ev0.elapsed_time(ev1) / 1000.0)
    value = world * B * args.steps / t_dev

    # ---- per-stage device times (separate instrumented pass over the same steps)
    ctx.enable_stage_timing(True)
    stages = {k: 0.0 for k in bl.STAGES}
    for _ in range(max(1, min(3, args.steps))):
        ctx.detect_landmarks(dev_frames, flat=True)
        for k, v in ctx.stage_times().items():
            stages[k] += v
    n_inst = max(1, min(3, args.steps))
    stages = {k: v / n_inst for k, v in stages.items()}
    ctx.enable_stage_timing(False)

    # ---- end-to-end through the public call with pinned host frames: H2D of every step's
    # frames and D2H of all its detections + landmarks inside the timed region
    e2e = None
    if not args.no_e2e:
        pinned = torch.from_numpy(frames).pin_memory()
        host = pinned.numpy()
        run_steps(host, max(1, args.warmup))
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n_faces = run_steps(host, args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(max(e0.elapsed_time(e1) / 1000.0, time.perf_counter() - t0))
        d2h = B * 4 + 12 + n_faces * (32 + 68 * 2 * 8)
        e2e = {"value": round(world * B * args.steps / t_e2e, 1), "unit": "frames/s",
               "h2d_bytes_per_step": B * W * H, "d2h_bytes_per_step": d2h,
               "api": f"bl_submit/bl_collect ({bl.MAX_IN_FLIGHT} batches in flight), pinned host frames"}

    # ---- roofline of the dominant stage
    alg = algorithmic_bytes_per_frame()
    peaks, peak_note = {}, "of fallback (B200_PROFILING.md: 6650 GB/s, 1590 bf16 TFLOP/s; MEASURED_PEAKS.json absent)"
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak_note = "of measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    f16_peak = float(peaks.get("bf16_tflops", 1590.0))  # dense fp16 = the bf16 rate
    traffic = {}
    try:  # ncu dram__bytes_read + write per frame of each stage's kernels (profiles/traffic.json)
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["bytes_per_frame"]
    except Exception:
        pass
    kern_ms = {k: stages[k] for k in ("pyramid", "gradhist", "features", "screen", "rescore", "nms", "ert")}
    dom = max(kern_ms, key=kern_ms.get)
    ert_bytes = faces_per_step * ERT_T * ERT_K * (68 * 2 * 8 + ERT_F * 48 + ERT_F * 2)
    bytes_stage = {"pyramid": alg["pyramid"] * B, "gradhist": alg["gradhist"] * B, "features": alg["features"] * B,
                   "screen": alg["screen"] * B, "ert": ert_bytes}
    per_stage = {}
    for k, ms in kern_ms.items():
        e = {"ms": round(ms, 3)}
        if k in bytes_stage and ms > 0:
            gbs = bytes_stage[k] / (ms / 1000.0) / 1e9
            e.update({"GB/s": round(gbs, 1), "frac_hbm": round(gbs / hbm_peak, 3)})
        if k in traffic:
            e["dram_GB_ncu"] = round(traffic[k] * B / 1e9, 3)
        per_stage[k] = e
    # secondary bounds (profiles/peaks_b200.json, measured on the box by tools/peaks.cu):
    # gradHist against the fp64 pipe, the ERT cascade against L2 read bandwidth
    try:
        sec = json.load(open(os.path.join(ROOT, "profiles", "peaks_b200.json")))
        if kern_ms["gradhist"] > 0:
            ops = GRADHIST_FP64_OPS * alg["gradhist_px"] * B / (kern_ms["gradhist"] / 1000.0) / 1e12
            per_stage["gradhist"].update({"fp64_Tops": round(ops, 2),
                                          "frac_fp64": round(ops / sec["fp64_add_tflops"], 3)})
        if kern_ms["ert"] > 0:
            l2 = ert_bytes / (kern_ms["ert"] / 1000.0) / 1e9
            per_stage["ert"].update({"frac_l2": round(l2 / sec["l2_read_gbs"], 3)})
    except Exception:
        pass
    if kern_ms["screen"] > 0:  # the tcgen05 screen: useful FLOPs (dense 10x10x31 x 5 filters)
        tfs = 2 * 5 * 3100 * alg["anchors"] * B / (kern_ms["screen"] / 1000.0) / 1e12
        per_stage["screen"].update({"TFLOP/s": round(tfs, 1), "frac_f16": round(tfs / f16_peak, 3)})
    ach = bytes_stage.get(dom, 0) / (kern_ms[dom] / 1000.0) / 1e9
    roofline = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(ach / hbm_peak, 3),
                "traffic": round(traffic[dom] * B / 1e9, 3) if dom in traffic else None,
                "traffic_unit": "GB per step (ncu dram__bytes_read+write.sum, profiles/traffic.json)",
                "peak_source": peak_note}
    roofline["kernel"] = dom
    if dom == "gradhist":  # what actually bounds it (ncu, profiles/r1v6_ncu_kernels.txt, DESIGN §5/§9)
        roofline["limiter"] = ("instruction issue: 62% issue-active at 16 warps/SM, ~108 instructions per level "
                               "pixel for the exact fp64 gradient/orientation/histogram (fp64 pipe: frac_fp64 in "
                               "stages_ms.gradhist)")

    # ---- CPU baseline (rank 0, N=1): the reference library on this box's cores
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(frames, det, ert, n=min(B, args.ref_frames * 2))

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_dev / args.steps * 1000.0, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{W}x{H} synthetic ring frames (u8), reference pattern detector (5 filters), "
                               f"ERT {ERT_T}x{ERT_K}xdepth{ERT_F} random-init 68 landmarks on every kept detection",
                   "frames_per_gpu_per_step": B, "global_batch": B * world, "faces_per_step_per_gpu": faces_per_step,
                   "parallelism": f"frame shards, {world} independent replicas, no collective",
                   "l2": f"inputs larger than L2 ({B * W * H / 1e6:.0f} MB u8 frames per step > 126 MB)"},
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk.summary(),
        "gpu_launches": int(launches * args.steps), "stages_ms": per_stage,
        "ms_per_step_wall": round(t_wall / args.steps * 1000.0, 3),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(frames, det, ert, n):
    """The UNMODIFIED reference (oracle/_ref) timed on this host: detect_faces + predict_landmarks
    on every kept detection, frame-parallel over all host threads (pipeline.cpp's scheme)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        from pyoracle import Reference
        ref = Reference()
        kind = "reference"
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "frames/s", "cores": 0, "kind": "unavailable", "sample": str(e)}
    threads = os.cpu_count() or 1
    sample = np.ascontiguousarray(frames[:n])
    ref.run_batch_u8(sample[:threads], det, ert, threads)  # warm-up (page-in, model build)
    t0 = time.perf_counter()
    reps, faces = 0, 0
    while True:  # ~10-30 s of CPU work: repeat the sample until >= 10 s wall
        f, counts, _ = ref.run_batch_u8(sample, det, ert, threads)
        faces += f
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= 10.0 or reps >= 200:
            break
    return {"value": round(n * reps / dt, 3), "unit": "frames/s", "cores": threads, "kind": kind,
            "sample": f"{n} distinct {W}x{H} frames x {reps} passes = {n * reps} frames, {faces} faces "
                      f"landmarked, {dt:.1f} s wall on {threads} threads"}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    det, ert = load_models()
    n = args.ref_frames
    frames = frames_for(0, n)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference
    ref = Reference()
    threads = os.cpu_count() or 1
    for _ in range(max(1, min(args.warmup, 1))):
        ref.run_batch_u8(frames[:threads], det, ert, threads)
    t0 = time.perf_counter()
    faces = 0
    for _ in range(args.steps):
        f, _, _ = ref.run_batch_u8(frames, det, ert, threads)
        faces += f
    dt = time.perf_counter() - t0
    v = n * args.steps / dt
    line = {
        "metric": METRIC, "value": round(v, 3), "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1000, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{W}x{H} synthetic ring frames (u8), reference pattern detector (5 filters), "
                               f"ERT {ERT_T}x{ERT_K}xdepth{ERT_F} random-init 68 landmarks on every kept detection",
                   "frames_per_step": n, "parallelism": f"frame-parallel std::threads x{threads} (host CPU)"},
        "cpu_baseline": {"value": round(v, 3), "unit": "frames/s", "cores": threads, "kind": "reference",
                         "sample": f"{n} frames per step x {args.steps} steps, {faces} faces landmarked"},
        "e2e": {"value": round(v, 3), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
