"""Multi-rank sampling logic on CPU (gloo, world_size 2): shot-range
sharding + the per-measurement count all-reduce. Each rank computes its
range with the CPU oracle's shot-keyed draws (keyed_draw is order-insensitive,
sampler.hpp:21-26), so the reduced counts must equal a single-process run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_03906_b200.distributed import shard_range


@pytest.mark.parametrize("total,world,tile", [(10_000_000, 8, 4096), (1, 2, 128), (4096, 3, 4096),
                                              (123_457, 4, 128), (0, 2, 64)])
def test_shard_range_partitions(total, world, tile):
    spans = [shard_range(total, world, r, tile) for r in range(world)]
    pos = 0
    for b, n in spans:
        assert b == pos or n == 0
        assert b % tile == 0 or n == 0
        pos = b + n if n else pos
    assert sum(n for _, n in spans) == total
    counts = [n for _, n in spans]
    assert max(counts) - min(counts) <= 2 * tile  # one extra tile + the ragged end


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, text, total, seed, tile, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2311_03906_b200 import run_initialization
    from paper_2311_03906_b200.distributed import all_reduce_counts, shard_range as sr

    init = run_initialization(text)
    port_ = oracle.Port()
    b, n = sr(total, world, rank, tile)
    S = port_.draw_assignments(init, n, seed, shot_begin=b)
    m = port_.sample(init.row_ptr, init.sym_idx, S, n)
    counts = torch.from_numpy(np.bitwise_count(m).sum(axis=1).astype(np.int64))
    all_reduce_counts(counts)
    q.put((rank, b, n, counts.numpy()))
    dist.destroy_process_group()


def test_gloo_two_rank_counts_match_single_process(port):
    from paper_2311_03906_b200 import circuits, run_initialization
    text = circuits.surface_code(3, 3, 0.01)
    total, seed, tile, world = 5000, 7, 256, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p_port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, p_port, text, total, seed, tile, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    init = run_initialization(text)
    S = port.draw_assignments(init, total, seed)
    m = port.sample(init.row_ptr, init.sym_idx, S, total)
    want = np.bitwise_count(m).sum(axis=1)
    for rank, b, n, counts in res:
        assert np.array_equal(counts, want), rank
    assert sorted((b, n) for _, b, n, _ in res)[0][0] == 0


class _FakeSampler:
    """CPU stand-in for Sampler: deterministic per-(global shot) outcomes, so
    the union of the ranks' shards equals one single-process run."""

    shot_tile = 64

    def __init__(self, n_meas):
        self.n_meas = n_meas

    def counts_for(self, begin, count, seed):
        shots = np.arange(begin, begin + count, dtype=np.int64)
        rows = np.arange(self.n_meas, dtype=np.int64)[:, None]
        bits = ((shots[None, :] * 2654435761 + rows * 40503 + seed) >> 7) & 1
        return bits.sum(axis=1)

    def sample(self, count, seed, shot_begin=0, out=None, counts=None):
        if counts is not None:
            counts += torch.from_numpy(self.counts_for(shot_begin, count, seed))
        return out


def _pipeline_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_03906_b200.distributed import CountPipeline, sample_sharded

    smp = _FakeSampler(5)
    total = 1000
    # sample_sharded: this rank's shard + the count all-reduce
    c = torch.zeros(5, dtype=torch.int64)
    b, n, _ = sample_sharded(smp, total, 3, counts=c)
    # bench's step loop: double-buffered async reduces, buffers reused
    seen = {}
    pipe = CountPipeline(5, "cpu", world,
                         on_reduced=lambda i, t: seen.__setitem__(i, t.clone().numpy()))
    for i in range(6):
        pipe.step(i, lambda cnt, i=i: smp.sample(n, 100 + i, shot_begin=b, counts=cnt),
                  last=i == 5)
    q.put((rank, b, n, c.numpy(), seen))
    dist.destroy_process_group()


def test_gloo_sample_sharded_and_step_pipeline():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p_port = _free_port()
    procs = [ctx.Process(target=_pipeline_worker, args=(r, world, p_port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    smp = _FakeSampler(5)
    total = 1000
    spans = sorted((b, n) for _, b, n, _, _ in res)
    assert spans[0][0] == 0 and sum(n for _, n in spans) == total
    want = smp.counts_for(0, total, 3)
    for rank, b, n, c, seen in res:
        assert np.array_equal(c, want), rank
        assert sorted(seen) == list(range(6))
        for i, got in seen.items():
            # each step's reduced counts = the sum over ranks of that step
            # only (the buffer is zeroed before reuse, nothing accumulates)
            want_i = sum(smp.counts_for(bb, nn, 100 + i) for bb, nn in spans)
            assert np.array_equal(got, want_i), (rank, i)


def _protocol_worker(rank, world, port, q):
    """bench.step_protocol with the bench's CountPipeline on gloo: the soak
    runs a rank-dependent number of times (rank 1's clock runs slow), yet
    every rank issues the same collectives, so nothing hangs and each step's
    reduce pairs with the same step on the other rank."""
    import time

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2311_03906_b200.distributed import CountPipeline

    smp = _FakeSampler(5)
    seen = {}
    pipe = CountPipeline(5, "cpu", world,
                         on_reduced=lambda i, t: seen.__setitem__(i, t.clone().numpy()))
    n_soak = [0]

    def soak():
        time.sleep(0.01 * (1 + 3 * rank))
        n_soak[0] += 1

    def step(i, last=False):
        pipe.step(i, lambda c: smp.sample(100, 100 + i, shot_begin=100 * rank, counts=c), last=last)

    t0 = time.perf_counter()
    marks = []  # (mark, steps reduced so far): the timed window holds exactly the 4 timed steps
    evs, wall = bench.step_protocol(step, soak, 3, 4, dist.barrier, lambda: None,
                                    lambda: time.perf_counter() - t0, lambda fn: fn(),
                                    on_timed=lambda k: marks.append((k, len(seen))))
    assert marks == [(0, 3), (1, 7)], marks
    q.put((rank, n_soak[0], len(evs), seen))
    dist.destroy_process_group()


def test_gloo_bench_step_protocol_ranks_agree():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_protocol_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    smp = _FakeSampler(5)
    assert res[0][1] != res[1][1]  # different soak counts ...
    for rank, _, n_ev, seen in res:  # ... same collectives: 3 warm-up + 4 timed steps
        assert n_ev == 4 and sorted(seen) == list(range(7))
        for i, got in seen.items():
            want = sum(smp.counts_for(100 * r, 100, 100 + i) for r in range(world))
            assert np.array_equal(got, want), (rank, i)
