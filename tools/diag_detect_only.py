import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
import paper_2006_00816_b200 as bl
det, ert = bench.load_models()
frames = bench.frames_for(0, 512)
dev = torch.from_numpy(frames).cuda()
ctx = bl.Context(0); ctx.upload_detector(det); ctx.upload_ert(ert)
stream = torch.cuda.current_stream(); ctx.set_stream(stream.cuda_stream)
def run(k, lm):
    pend = [ctx.submit(dev, landmarks=lm) for _ in range(3)]
    issued = 3
    while pend:
        ctx.collect(pend.pop(0)); 
        if issued < k: pend.append(ctx.submit(dev, landmarks=lm)); issued += 1
for lm in (True, False, True, False):
    run(5, lm); torch.cuda.synchronize()
    t0 = time.perf_counter(); run(20, lm); torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"landmarks={lm}: {t/20*1000:.2f} ms/step, {512*20/t:.0f} fps")
