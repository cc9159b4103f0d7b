"""Diagnose e2e vs device-resident throughput: raw pinned H2D bandwidth and per-phase timing."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2006_00816_b200 as bl

det, ert = bench.load_models()
frames = bench.frames_for(0, 512)
pinned = torch.from_numpy(frames).pin_memory()
dev = torch.empty_like(pinned, device="cuda")
for _ in range(3):
    dev.copy_(pinned, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    dev.copy_(pinned, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"pinned H2D {pinned.numel()/1e6:.0f} MB: {ms:.2f} ms = {pinned.numel()/ms/1e6:.1f} GB/s")
ctx = bl.Context(0); ctx.upload_detector(det); ctx.upload_ert(ert)
host = pinned.numpy()
for src, name in [(dev, "device"), (host, "host")]:
    ctx.detect_landmarks(src, flat=True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5): ctx.detect_landmarks(src, flat=True)
    t1 = time.perf_counter()
    print(f"sync {name}: {(t1-t0)/5*1000:.2f} ms/step")
    p = ctx.submit(src); t0 = time.perf_counter()
    for i in range(10):
        q = ctx.submit(src); ctx.collect(p); p = q
    ctx.collect(p); t1 = time.perf_counter()
    print(f"pipelined {name}: {(t1-t0)/11*1000:.2f} ms/step")
