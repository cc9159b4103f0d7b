"""C2 throughput (16 x 320x240 frames per batch, device-resident, 4 in flight) with and without
the landmark cascade: how much of the batch interval the cascade costs."""
import os
import sys

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
fr = torch.from_numpy(bench.tiled_frames(16, 320, 240)).cuda()
for lm in (True, False, True, False):
    bench.pipelined(ctx, bl, fr, 20, landmarks=lm)
    t, _, _ = bench.timed(torch, stream, lambda: bench.pipelined(ctx, bl, fr, 400, landmarks=lm))
    print("landmarks" if lm else "detect-only", round(16 * 400 / t, 1), "frames/s", round(t / 400 * 1e6, 1), "us/batch")
