"""bl_run throughput (decode + detect + best-face landmarks + EAR), several timed repeats:
python tools/run_rate.py [n_frames] [batch]"""
import os
import shutil
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2006_00816_b200 as bl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
det, ert = bench.load_models()
ctx = bl.Context(0)
ctx.upload_detector(det)
ctx.upload_ert(ert)
d = tempfile.mkdtemp(prefix="bl_run_")
try:
    for i, f in enumerate(bench.tiled_frames(n, bench.W, bench.H, distinct=32, seed=91)):
        bl.write_pgm(os.path.join(d, f"frame_{i:06d}.pgm"), f)
    ctx.run(d, 30.0, batch_size=batch)
    rates = []
    for _ in range(6):
        t0 = time.perf_counter()
        ctx.run(d, 30.0, batch_size=batch)
        rates.append(n / (time.perf_counter() - t0))
    print("run frames/s", [round(r) for r in rates])
finally:
    shutil.rmtree(d, ignore_errors=True)
