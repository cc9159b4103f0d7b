"""Device-resident vs end-to-end (pinned host frames through submit/collect) rate at the bench
batch, with and without the landmark cascade: where the e2e gap comes from."""
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
B, W_, H_ = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (512, 640, 480)))
fr = bench.frames_range(0, B, W_, H_) if (W_, H_) == (640, 480) else bench.tiled_frames(B, W_, H_)
dev = torch.from_numpy(fr).cuda()
host = torch.from_numpy(fr).pin_memory().numpy()
for lm in (True, False):
    for name, src in (("device", dev), ("e2e", host)):
        bench.pipelined(ctx, bl, src, 4, landmarks=lm)
        k = max(30, int(0.8e9 / (B * W_ * H_)))
        t, tw, _ = bench.timed(torch, stream, lambda: bench.pipelined(ctx, bl, src, k, landmarks=lm))
        print("landmarks" if lm else "detect-only", name, round(B * k / max(t, tw), 1), "frames/s")
