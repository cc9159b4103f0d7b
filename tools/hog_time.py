"""gradHist stage time at the bench batch (HOG_BATCH, default 1024 x 640x480 frames, device-resident), detection
only, with a large face capacity so timing experiments that break results still run.
    BL_LIBRARY=... python tools/hog_time.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2006_00816_b200 as bl  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
det, ert = bench.load_models()
ctx = bl.Context(0)
ctx.upload_detector(det)
ctx.set_face_capacity(4096)
frames = torch.from_numpy(bench.frames_range(0, int(os.environ.get("HOG_BATCH", "1024")))).cuda()
ctx.detect(frames, flat=True)
ctx.enable_stage_timing(True)
acc = {}
for _ in range(reps):
    try:
        ctx.detect(frames, flat=True, cap=1 << 24)
    except Exception as e:  # noqa: BLE001
        print("detect:", str(e)[:120])
    for k, v in ctx.stage_times().items():
        acc[k] = acc.get(k, 0.0) + v / reps
print(os.environ.get("TAG", "?"), " ".join(f"{k}={v:.4f}" for k, v in acc.items()))
