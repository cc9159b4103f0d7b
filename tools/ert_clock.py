"""Per-phase clock64 totals of the latency ERT kernels on one face (BL_WD_CLOCK build), cold
then warm:  BL_LIBRARY=variants/wdclock/libblinkline_b200.so BL_ERT=wide [BL_ERT_CL=4] python tools/ert_clock.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2006_00816_b200 as bl  # noqa: E402

det, ert = bench.load_models()
c = bl.Context(0)
c.upload_ert(ert)
f = bench.frames_range(0, 1)
for _ in range(3):
    c.landmarks(f, [0], [[200, 100, 240, 240]])
    c.synchronize()
