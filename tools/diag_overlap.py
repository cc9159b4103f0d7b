import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2006_00816_b200 as bl

det, ert = bench.load_models()
frames = bench.frames_for(0, 512)
pinned = torch.from_numpy(frames).pin_memory()
dev = pinned.cuda()
dst = torch.empty_like(dev)
ctx = bl.Context(0); ctx.upload_detector(det); ctx.upload_ert(ert)
cs = torch.cuda.Stream()
ctx.detect_landmarks(dev, flat=True); torch.cuda.synchronize()
for label, copy in [("compute only", False), ("compute + concurrent H2D", True)]:
    t0 = time.perf_counter()
    for _ in range(5):
        if copy:
            with torch.cuda.stream(cs):
                dst.copy_(pinned, non_blocking=True)
        ctx.detect_landmarks(dev, flat=True)
    torch.cuda.synchronize()
    print(label, f"{(time.perf_counter()-t0)/5*1000:.2f} ms/step")
# the same with the copy issued as 8 chunks
t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(cs):
        for c in range(8):
            dst[c*64:(c+1)*64].copy_(pinned[c*64:(c+1)*64], non_blocking=True)
    ctx.detect_landmarks(dev, flat=True)
torch.cuda.synchronize()
print("compute + chunked H2D", f"{(time.perf_counter()-t0)/5*1000:.2f} ms/step")
