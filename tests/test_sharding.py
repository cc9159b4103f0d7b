"""Multi-GPU frame sharding, exercised on CPU with the gloo backend at world_size 2: shards
partition the batch, per-rank results come back in global frame order, and the timing rule
takes the max over ranks.  (frames are independent, no data-path collective.)"""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2006_00816_b200.sharding import shard_range


def test_shard_range_partitions():
    for n in [0, 1, 7, 16, 513]:
        for world in [1, 2, 3, 8]:
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch.distributed as dist

    from paper_2006_00816_b200.sharding import gather_in_frame_order, max_over_ranks
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = shard_range(n, rank, world)
    # stand-in per-frame result: (frame index, detections) as the bench's ranks produce
    local = [(i, [i * 10 + k for k in range(i % 3)]) for i in range(b, e)]
    full = gather_in_frame_order(local, rank, world, n)
    t = max_over_ranks(1.0 + rank)
    if rank == 0:
        q.put((full, t))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_gather_and_max():
    n, world = 11, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert [f[0] for f in full] == list(range(n))
    assert full[5] == (5, [50, 51, 52][:5 % 3])
    assert t == 2.0


def _sharded_worker(rank, world, port, n, q):
    """One rank of the real shard -> run -> gather path (sharding.run_sharded), with the CPU
    oracle's detect_faces as the per-frame stage (no GPU here)."""
    import numpy as np
    import torch.distributed as dist

    from paper_2006_00816_b200.sharding import run_sharded
    from paper_2006_00816_b200.synthetic import ring_frames_range
    from pyoracle import Oracle

    import bench
    det, _ = bench.load_models()
    orc = Oracle()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def process(frames):
        return [[tuple(int(d[k]) for k in ("x", "y", "w", "h")) + (float(d["score"]),)
                 for d in orc.detect_faces(f.astype(np.float64), det)] for f in frames]

    b, e, local, full = run_sharded(n, rank, world, lambda b, e: ring_frames_range(b, e, 320, 240, seed=9), process)
    if rank == 0:
        q.put((b, e, full))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_real_shard_run_gather(oracle):
    """world_size 2: each rank builds its own shard of a global synthetic sequence, runs the
    per-frame stage and the results come back on rank 0 in global frame order, identical to
    one process running the whole sequence."""
    import numpy as np

    import bench
    from paper_2006_00816_b200.synthetic import ring_frames_range
    n, world = 7, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    b, e, full = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert (b, e) == (0, 4)
    det, _ = bench.load_models()
    frames = ring_frames_range(0, n, 320, 240, seed=9)
    want = [[tuple(int(d[k]) for k in ("x", "y", "w", "h")) + (float(d["score"]),)
             for d in oracle.detect_faces(f.astype(np.float64), det)] for f in frames]
    assert full == want
    assert sum(len(x) for x in full) > 0


def test_ring_frames_range_is_shard_independent():
    import numpy as np

    from paper_2006_00816_b200.synthetic import ring_frames_range
    whole = ring_frames_range(0, 5, 96, 80)
    parts = np.concatenate([ring_frames_range(0, 2, 96, 80), ring_frames_range(2, 5, 96, 80)])
    assert np.array_equal(whole, parts)


def test_bench_launcher_spawns_ranks():
    """bench.py --gpus N without WORLD_SIZE launches N ranks itself (RANK / LOCAL_RANK /
    WORLD_SIZE / MASTER_*), which rendezvous; here over gloo with --launcher-selftest."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "3", "--launcher-selftest"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 3
    assert sorted(r["rank"] for r in line["ranks"]) == [0, 1, 2]
    assert [r["local_rank"] for r in sorted(line["ranks"], key=lambda r: r["rank"])] == [0, 1, 2]
    assert len({r["pid"] for r in line["ranks"]}) == 3


def test_reference_arm_does_not_map_the_gpu_library():
    """The --impl reference arm times the reference library alone: the process never maps
    libblinkline_b200.so (importing the package as a side effect tainted it)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','0','--batch','8'];"
            f"sys.path.insert(0, {root!r}); import bench; bench.main();"
            "m=open('/proc/self/maps').read(); print('OURS' if 'libblinkline_b200' in m else 'CLEAN',"
            " 'REF' if 'libblinkline_ref' in m else 'NOREF')")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr
    last = out.stdout.strip().splitlines()[-1]
    assert last == "CLEAN REF", out.stdout
