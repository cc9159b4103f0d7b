"""Device-resident frames/s at the bench batch (512 x 640x480) with and without the landmark
cascade (4 batches in flight through submit/collect): the cascade's marginal cost per step."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2006_00816_b200 as bl  # noqa: E402

det, ert = bench.load_models()
ctx = bl.Context(0)
ctx.upload_detector(det)
ctx.upload_ert(ert)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
fr = torch.from_numpy(bench.frames_range(0, 512)).cuda()
for lm in (True, False, True, False):
    bench.pipelined(ctx, bl, fr, 4, landmarks=lm)
    t, _, _ = bench.timed(torch, stream, lambda: bench.pipelined(ctx, bl, fr, 20, landmarks=lm))
    print("landmarks" if lm else "detect-only", round(512 * 20 / t, 1), "frames/s", round(t / 20 * 1000, 3), "ms/step")
