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
