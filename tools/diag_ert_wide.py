"""Landmark cascade latency vs face count: k_ert_wide (face per CTA) against k_ert_cascade
(kFcFaces faces per CTA).  GPU box:  BL_ERT=wide python tools/diag_ert_wide.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2006_00816_b200 as bl
from paper_2006_00816_b200.synthetic import ring_frames_np

det, ert = bench.load_models()
ctx = bl.Context(0); ctx.upload_ert(ert)
frames = ring_frames_np(1, 640, 480, seed=5)
rng = np.random.default_rng(3)
out = []
for nf in (4, 16, 64, 148, 296, 600, 1200, 2400):
    side = rng.integers(120, 280, nf)
    boxes = np.stack([rng.integers(0, 640 - side), rng.integers(0, 480 - side), side, side], 1).astype(np.int32)
    fob = np.zeros(nf, np.int32)
    ctx.landmarks(frames, fob, boxes)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); ctx.landmarks(frames, fob, boxes); ts.append(time.perf_counter() - t0)
    out.append(f"{nf}:{np.median(ts)*1e3:.3f}")
print(os.environ.get("BL_ERT", "auto"), os.environ.get("BL_LIBRARY", "main").split("/")[-2] if "BL_LIBRARY" in os.environ else "main", " ".join(out))
