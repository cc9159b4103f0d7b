"""C2 (320x240 x16) latency breakdown on the GPU box: stage times, host cost of submit/collect,
and throughput at 1..4 batches in flight."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2006_00816_b200 as bl
from paper_2006_00816_b200.synthetic import ring_frames_np

det, ert = bench.load_models()
ctx = bl.Context(0); ctx.upload_detector(det); ctx.upload_ert(ert)
for (w, h, b) in [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]] or ((640, 480, 1), (320, 240, 16), (640, 480, 512)):
    frames = ring_frames_np(b, w, h, seed=77)
    dev = torch.from_numpy(frames).cuda()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        ctx.detect_landmarks(dev, flat=True)
    ctx.enable_stage_timing(True)
    ctx.detect_landmarks(dev, flat=True)
    print(w, h, b, "stages", {k: round(v, 3) for k, v in ctx.stage_times().items()})
    ctx.enable_stage_timing(False)
    torch.cuda.synchronize()
    # host cost of one submit and one collect
    ts, tc = [], []
    for _ in range(20):
        t0 = time.perf_counter(); t = ctx.submit(dev, landmarks=True); t1 = time.perf_counter()
        torch.cuda.synchronize(); t2 = time.perf_counter(); ctx.collect(t, flat=True); t3 = time.perf_counter()
        ts.append(t1 - t0); tc.append(t3 - t2)
    print("  host submit ms", round(np.median(ts) * 1e3, 3), "collect (after sync) ms", round(np.median(tc) * 1e3, 3))
    for inflight in (1, 2, 3, 4):
        n = 60
        torch.cuda.synchronize(); t0 = time.perf_counter()
        pend = []
        for i in range(n):
            pend.append(ctx.submit(dev, landmarks=True))
            if len(pend) >= inflight:
                ctx.collect(pend.pop(0), flat=True)
        while pend:
            ctx.collect(pend.pop(0), flat=True)
        dt = (time.perf_counter() - t0) / n
        print(f"  in flight {inflight}: {dt*1e3:.3f} ms/batch, {b/dt:.0f} frames/s")
