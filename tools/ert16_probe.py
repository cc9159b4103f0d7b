import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, bench, paper_2006_00816_b200 as bl
from paper_2006_00816_b200.synthetic import ring_frames_np
det, ert = bench.load_models()
ctx = bl.Context(0); ctx.upload_ert(ert)
frames = ring_frames_np(1, 640, 480, seed=5)
rng = np.random.default_rng(3); nf = 16
side = rng.integers(120, 280, nf)
boxes = np.stack([rng.integers(0, 640 - side), rng.integers(0, 480 - side), side, side], 1).astype(np.int32)
for _ in range(3): ctx.landmarks(frames, np.zeros(nf, np.int32), boxes)
