"""How often do faces of one ERT CTA (consecutive kept detections) pick the same leaf?
Measures the leaf-row reuse a per-CTA cache could exploit on the bench workload."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import bench
import paper_2006_00816_b200 as bl

det, ert = bench.load_models()
frames = bench.frames_for(0, 64)
ctx = bl.Context(0)
ctx.upload_detector(det)
ctx.upload_ert(ert)
dets, _ = ctx.detect_landmarks(frames)
ff, bx = [], []
for i, d in enumerate(dets):
    for r in d:
        ff.append(i)
        bx.append([r["x"], r["y"], r["w"], r["h"]])
ff = np.array(ff, np.int32)
bx = np.array(bx, np.int32)
_, leaves = ctx.landmarks(frames, ff, bx, want_leaves=True)
n = len(ff)
print("faces", n, "per frame", n / len(frames))
for g in (2, 4, 8, 16, 32):
    distinct = 0
    for a in range(0, n - g + 1, g):
        L = leaves[a:a + g]  # g x (T*K)
        distinct += sum(len(np.unique(L[:, j])) for j in range(L.shape[1]))
    groups = (n // g)
    print(f"group {g}: leaf rows per face {distinct / (groups * g * leaves.shape[1]):.3f}")
