"""Frame sharding across GPUs: frames are independent, so a batch is split
into contiguous per-rank shards, each rank runs the whole hot path on its shard with its own
model replica, and results are gathered on the host in frame order (the order-restoring
scheme of the reference's pipeline, pipeline.cpp:302-303).  No collective touches the data
path; torch.distributed is used only for the result gather and for max-over-ranks timing."""

from __future__ import annotations


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) frame range of `rank`; shard sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def gather_in_frame_order(local_results: list, rank: int, world: int, n_total: int, group=None):
    """Collect per-frame results from every rank onto rank 0, restoring global frame order.
    Returns the full list on rank 0 and None elsewhere."""
    import torch.distributed as dist

    if world == 1:
        return list(local_results)
    begin, end = shard_range(n_total, rank, world)
    if len(local_results) != end - begin:
        raise ValueError("local result count does not match the shard")
    parts = [None] * world if rank == 0 else None
    dist.gather_object((begin, local_results), parts, dst=0, group=group)
    if rank != 0:
        return None
    out = [None] * n_total
    for b, res in parts:
        out[b:b + len(res)] = res
    return out


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (the bench's timing rule: the job is as slow as its slowest rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def run_sharded(n_total: int, rank: int, world: int, make_frames, process, group=None):
    """shard -> run -> gather: this rank builds frames [begin, end) of the global batch with
    ``make_frames(begin, end)``, runs ``process(frames)`` (a list with one result per frame) and
    the per-frame results are gathered onto rank 0 in global frame order.  Returns
    (begin, end, local results, gathered list on rank 0 / None elsewhere)."""
    begin, end = shard_range(n_total, rank, world)
    local = list(process(make_frames(begin, end)))
    if len(local) != end - begin:
        raise ValueError("process() must return one result per frame")
    return begin, end, local, gather_in_frame_order(local, rank, world, n_total, group)
