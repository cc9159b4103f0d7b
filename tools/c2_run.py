"""C2 batches (16 x 320x240 frames) through detect + landmarks, a few times -- for ncu launch
lists of the small-batch kernels:  ncu --metrics gpu__time_duration.sum python tools/c2_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2006_00816_b200 as bl  # noqa: E402

det, ert = bench.load_models()
ctx = bl.Context(0)
ctx.upload_detector(det)
ctx.upload_ert(ert)
fr = bench.tiled_frames(16, 320, 240)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    d, c, l = ctx.detect_landmarks(fr, flat=True)
print("faces", len(d))
