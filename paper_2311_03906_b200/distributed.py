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


class CountPipeline:
    """Per-step count reduction, double-buffered (the bench's step loop).

    Step i samples into buffer i % 2 (zeroed first: the sampler adds into it)
    and starts an asynchronous all-reduce of it; step i+1 samples into the
    other buffer while that reduce runs. A buffer's previous reduce is waited
    for before the buffer is reused, and `on_reduced(step, counts)` then sees
    the step's global counts. `flush()` waits for everything in flight.
    """

    def __init__(self, n: int, device, world: int, group=None, on_reduced=None):
        import torch
        self.world, self.group, self.on_reduced = world, group, on_reduced
        self.bufs = [torch.zeros(n, dtype=torch.int64, device=device) for _ in range(2)]
        self.pending = [None, None]  # (work handle or None, step index)

    def _finish(self, b: int):
        work, i = self.pending[b]
        if work is not None:
            work.wait()
        self.pending[b] = None
        if self.on_reduced is not None:
            self.on_reduced(i, self.bufs[b])

    def step(self, i: int, sample_into, last: bool = False):
        """sample_into(counts) adds this rank's step-i counts into `counts`."""
        import torch.distributed as dist
        b = i % 2
        if self.pending[b] is not None:
            self._finish(b)
        buf = self.bufs[b]
        buf.zero_()
        sample_into(buf)
        work = None
        if self.world > 1:
            work = dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        self.pending[b] = (work, i)
        if last:
            self.flush()
        return buf

    def flush(self):
        for b in sorted(range(2), key=lambda k: -1 if self.pending[k] is None
                        else self.pending[k][1]):
            if self.pending[b] is not None:
                self._finish(b)
