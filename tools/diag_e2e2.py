import sys, os, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
import paper_2006_00816_b200 as bl
det, ert = bench.load_models()
frames = bench.frames_for(0, 512)
pinned = torch.from_numpy(frames).pin_memory()
dev = pinned.cuda()
ctx = bl.Context(0); ctx.upload_detector(det); ctx.upload_ert(ert)
stream = torch.cuda.current_stream(); ctx.set_stream(stream.cuda_stream)
host = pinned.numpy()
def run(src, k):
    p = ctx.submit(src)
    for i in range(k):
        q = ctx.submit(src) if i + 1 < k else None
        ctx.collect(p); p = q
for name, src in [("device", dev), ("host", host), ("device", dev), ("host", host)]:
    run(src, 3); torch.cuda.synchronize()
    t0 = time.perf_counter(); run(src, 20); torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"{name}: {t/20*1000:.2f} ms/step wall, {512*20/t:.0f} fps")
# host-side cost of one submit while GPU is busy
p = ctx.submit(host); t0 = time.perf_counter(); q = ctx.submit(host); t1 = time.perf_counter()
ctx.collect(p); ctx.collect(q)
print(f"submit host time {1000*(t1-t0):.3f} ms")
t0 = time.perf_counter(); p = ctx.submit(dev); t1 = time.perf_counter(); ctx.collect(p); t2 = time.perf_counter()
print(f"submit {1000*(t1-t0):.3f} ms, collect {1000*(t2-t1):.3f} ms")
