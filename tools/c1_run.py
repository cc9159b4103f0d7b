"""One 640x480 frame per batch through detect + landmarks (the C1 workload), a few times --
for ncu captures of the small-batch kernels:  ncu -k regex:k_nms python tools/c1_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2006_00816_b200 as bl  # noqa: E402

det, ert = bench.load_models()
ctx = bl.Context(0)
ctx.upload_detector(det)
ctx.upload_ert(ert)
fr = bench.frames_range(0, 1)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    d, c, l = ctx.detect_landmarks(fr, flat=True)
print("faces", len(d))
