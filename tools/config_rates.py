"""Throughput of the BASELINE.json configurations beyond the bench line (GPU box, 1 GPU).

C2 320x240 x16, C3 1280x720 x64, C5 1920x1080 x256 (detect + 68 landmarks on every kept face,
frames resident in HBM, bl.MAX_IN_FLIGHT batches in flight through bl_submit / bl_collect) and C4 (landmarks
only: 10k boxes through the 15x500xdepth-4 cascade).  The reference CPU path is timed beside
each on a bounded sample with all host threads.  One JSON line per config on stdout:
    python tools/config_rates.py > profiles/r1v6_config_rates.jsonl"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2006_00816_b200 as bl  # noqa: E402
from paper_2006_00816_b200.synthetic import ring_frames_np  # noqa: E402


def device_rate(ctx, frames, steps=40, warmup=20):
    # steady state: enough batches that the 4-deep pipeline's fill / drain stays small (bench.py)
    steps = max(steps, int(0.8e9 / frames.size))
    dev = torch.from_numpy(frames).cuda()
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    def run(k):
        pend, issued, faces = [], 0, 0
        while issued < min(k, bl.MAX_IN_FLIGHT):
            pend.append(ctx.submit(dev, landmarks=True))
            issued += 1
        while pend:
            _, counts, _ = ctx.collect(pend.pop(0), flat=True)
            faces += int(np.sum(counts))
            if issued < k:
                pend.append(ctx.submit(dev, landmarks=True))
                issued += 1
        return faces

    run(warmup)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    faces = run(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1000.0
    return len(frames) * steps / t, faces / steps, t / steps * 1000.0


def cpu_rate(ref, frames, det, ert, budget_s=8.0):
    threads = os.cpu_count() or 1
    ref.run_batch_u8(frames[:min(len(frames), threads)], det, ert, threads)  # warm-up
    n, t0, done = 0, time.perf_counter(), 0
    while time.perf_counter() - t0 < budget_s:
        chunk = frames[done % len(frames):][:threads]
        ref.run_batch_u8(chunk, det, ert, threads)
        n += len(chunk)
        done += len(chunk)
    return n / (time.perf_counter() - t0), threads, n


def main():
    from pyoracle import Reference
    det, ert = bench.load_models()
    ref = Reference()
    ctx = bl.Context(0)
    ctx.upload_detector(det)
    ctx.upload_ert(ert)
    for name, w, h, b in (("C2", 320, 240, 16), ("C3", 1280, 720, 64), ("C5", 1920, 1080, 256)):
        frames = ring_frames_np(b, w, h, seed=77)
        fps, faces, ms = device_rate(ctx, frames)
        cfps, cores, nsample = cpu_rate(ref, frames, det, ert)
        print(json.dumps({"config": name, "frames": f"{w}x{h} x{b}", "frames_per_s": round(fps, 1),
                          "ms_per_batch": round(ms, 3), "faces_per_batch": faces,
                          "cpu_reference_frames_per_s": round(cfps, 2), "cpu_cores": cores,
                          "cpu_sample_frames": nsample, "speedup": round(fps / cfps, 1)}), flush=True)
    # C4: landmarks only, 10k boxes in one 640x480 frame
    r = np.random.default_rng(405)
    n = 10000
    side = r.integers(120, 280, n)
    boxes = np.stack([r.integers(0, 640 - side + 1), r.integers(0, 480 - side + 1), side, side], 1).astype(np.int32)
    img = np.floor(np.random.default_rng(404).uniform(0, 256, (480, 640))).astype(np.uint8)
    ff = np.zeros(n, np.int32)
    ctx.landmarks(img, ff, boxes)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        ctx.landmarks(img, ff, boxes)
    t = (time.perf_counter() - t0) / reps
    # reference: a bounded sample of the boxes through predict_landmarks on all threads
    k = 2000
    threads = os.cpu_count() or 1
    ref.landmarks_batch_u8(img[None], ff[:threads], boxes[:threads], ert, threads)  # warm-up
    tc = time.perf_counter()
    ref.landmarks_batch_u8(img[None], ff[:k], boxes[:k], ert, threads)
    tcpu = time.perf_counter() - tc
    print(json.dumps({"config": "C4", "boxes": n, "boxes_per_s": round(n / t, 1), "ms_per_10k": round(t * 1000, 3),
                      "timing": "wall clock incl. host<->device copies of boxes and landmarks",
                      "cpu_reference_boxes_per_s": round(k / tcpu, 1), "cpu_cores": threads,
                      "cpu_sample_boxes": k, "speedup": round((n / t) / (k / tcpu), 1)}), flush=True)


if __name__ == "__main__":
    main()
