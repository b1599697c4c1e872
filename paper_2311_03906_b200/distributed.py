"""Multi-GPU plumbing for the sampler: shot-range sharding + count reduction.

Shots are independent, so a run of N shots on G GPUs is G disjoint, tile-
aligned global shot ranges. Random streams are keyed by the
global shot tile, so the union of the per-rank records is bit-identical to a
single-GPU run. The only exchange is one all-reduce of per-measurement flip
counts (u64 -> int64 tensor) — NCCL over NVLink/NVSwitch on GPUs, gloo in
the CPU tests.
"""
from __future__ import annotations


def shard_range(total_shots: int, world: int, rank: int, tile: int) -> tuple[int, int]:
    """Contiguous, tile-aligned [begin, begin + count) of rank `rank`.

    Whole tiles are dealt out as evenly as possible (ranks differ by at most
    one tile); the last rank absorbs the ragged end.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if tile < 1:
        raise ValueError("tile must be positive")
    n_tiles = -(-total_shots // tile)
    base, extra = divmod(n_tiles, world)
    t0 = rank * base + min(rank, extra)
    t1 = t0 + base + (1 if rank < extra else 0)
    begin = min(t0 * tile, total_shots)
    end = min(t1 * tile, total_shots)
    return begin, end - begin


def all_reduce_counts(counts, group=None):
    """Sum per-measurement counts over all ranks in place (the one collective)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def sample_sharded(sampler, total_shots: int, seed: int, out=None, counts=None, group=None):
    """This rank's share of a global sampling run; returns (begin, count, out)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    begin, count = shard_range(total_shots, world, rank, sampler.shot_tile)
    if count:
        out = sampler.sample(count, seed, shot_begin=begin, out=out, counts=counts)
    if counts is not None:
        all_reduce_counts(counts, group)
    return begin, count, out
