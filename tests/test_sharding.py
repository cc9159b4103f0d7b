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
