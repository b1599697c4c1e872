"""K5 column sampler (k5_columns.cu) for dense M_sym: records == M_sym . S of
its own draw (bit-exact), == the CPU oracle on that S, invariant to how the
shot range is split, with the channel pmfs intact."""
import os

import numpy as np
import pytest

from paper_2311_03906_b200 import circuits as CI
from paper_2311_03906_b200 import run_initialization
from paper_2311_03906_b200.sampler import GROUP_DTYPE, InitResult

pytestmark = pytest.mark.gpu


def host(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.fixture
def force_k5():
    os.environ["SP_K5"] = "1"
    yield
    del os.environ["SP_K5"]


def mixed_dense_model(m, v, dens, seed):
    """Random dense M_sym over s0 + Bernoulli / DEPOLARIZE1 / DEPOLARIZE2
    groups (some dead), with s0 in a few rows and one p = 1 channel."""
    rng = np.random.default_rng(seed)
    groups, sym = [(0, 0.0, 0, 1)], 1
    while sym < v:
        kind = rng.integers(0, 4)
        if kind == 0:
            groups.append((1, float(rng.choice([1e-3, 0.02, 0.2])), sym, 1)); sym += 1
        elif kind == 1 and sym + 2 <= v:
            groups.append((3, float(rng.choice([1e-3, 0.05])), sym, 2)); sym += 2
        elif kind == 2 and sym + 4 <= v:
            groups.append((4, float(rng.choice([1e-3, 0.1])), sym, 4)); sym += 4
        else:
            groups.append((1, 1.0, sym, 1)); sym += 1
    g = np.zeros(len(groups), dtype=GROUP_DTYPE)
    for i, (d, p, f, a) in enumerate(groups):
        g[i]["dist"], g[i]["param"], g[i]["first_symbol"], g[i]["arity"] = d, p, f, a
    bits = rng.random((m, sym)) < dens
    bits[:, sym - sym // 10:] = False          # a tail of dead symbols
    bits[:, 0] = rng.random(m) < 0.2            # s0 in some rows
    rows = [np.nonzero(r)[0].astype(np.uint32) for r in bits]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.uint64)
    return InitResult(0, sym, rp, np.concatenate(rows).astype(np.uint32), g)


@pytest.mark.parametrize("m,v,n", [(300, 400, 5000), (1000, 900, 4096 + 77), (40, 150, 33)])
def test_k5_records_equal_product_of_its_draws(gpu_sampler_factory, port, force_k5, m, v, n):
    model = mixed_dense_model(m, v, 0.3, seed=m + v)
    s = gpu_sampler_factory(model)
    assert s.plan_info()["fused_ok"] == 2  # K5
    for seed in (1, 99):
        out = s.sample(n, seed)
        S = s.draw_assignments(n, seed)
        assert np.array_equal(host(out), host(s.sample_given(S, n))), seed
        assert np.array_equal(host(out), port.sample(model.row_ptr, model.sym_idx, host(S), n))


def test_k5_split_and_counts(gpu_sampler_factory, force_k5):
    import torch
    model = mixed_dense_model(500, 600, 0.4, seed=5)
    s = gpu_sampler_factory(model)
    T = s.shot_tile
    n = 6 * T
    whole = host(s.sample(n, 7))
    a = host(s.sample(3 * T, 7))
    b = host(s.sample(3 * T, 7, shot_begin=3 * T))
    assert np.array_equal(whole[:, : a.shape[1]], a)
    assert np.array_equal(whole[:, a.shape[1]:], b)
    counts = torch.zeros(model.n_meas, dtype=torch.int64, device="cuda")
    s.sample(n, 7, counts=counts)
    pc = np.unpackbits(whole.view(np.uint8), axis=1).sum(axis=1)
    assert np.array_equal(counts.cpu().numpy(), pc)


def test_k5_chosen_for_cfg5_density_half():
    """The planner picks K5 by itself for a dense M_sym with frequent faults."""
    from paper_2311_03906_b200 import Sampler
    model = CI.random_msym_model(2000, 20000, 0.5, 1e-2, seed=3)
    s = Sampler(model)
    assert s.plan_info()["fused_ok"] == 2


def test_k5_pattern_marginals_1M(gpu_sampler_factory, force_k5):
    """K5's streams keep the channel pmfs (DEPOLARIZE1: p/3 each pattern,
    DEPOLARIZE2: p/15, Bernoulli p) at 5 sigma."""
    N = 1_000_000
    model = mixed_dense_model(200, 300, 0.3, seed=11)
    s = gpu_sampler_factory(model)
    S = host(s.draw_assignments(N, 3))
    tail = N % 64
    valid = np.full(S.shape[1], ~np.uint64(0), dtype=np.uint64)
    if tail:
        valid[-1] = np.uint64((1 << tail) - 1)
    bad = []
    for gi in range(1, len(model.groups)):
        d, p, f = (int(model.groups["dist"][gi]), float(model.groups["param"][gi]),
                   int(model.groups["first_symbol"][gi]))
        arity = {1: 1, 3: 2, 4: 4}[d]
        npat = (1 << arity) - 1
        for pat in range(1, npat + 1):
            w = valid.copy()
            for b in range(arity):
                w &= S[f + b] if (pat >> b) & 1 else ~S[f + b]
            q = p if d == 1 else p / npat
            hits = int(np.bitwise_count(w).sum())
            sd = np.sqrt(max(q * (1 - q), 1e-300) / N)
            if abs(hits / N - q) > 5 * sd + 1e-12:
                bad.append((gi, d, p, pat, hits / N))
    assert not bad, bad


def test_k5_host_path_and_tiled(gpu_sampler_factory, port, force_k5):
    """sp_sample_to_host serves a K5 model through the same sampler as
    sp_sample (its b8 bytes equal the encoded records), and the tiled layout,
    which only the fused kernel produces, is refused."""
    from paper_2311_03906_b200._native import SymphaseError
    model = mixed_dense_model(150, 300, 0.3, seed=9)
    s = gpu_sampler_factory(model)
    assert s.plan_info()["fused_ok"] == 2
    n = 3000
    out = s.sample(n, 4)
    want = s.encode(out, n, "b8").cpu().numpy().tobytes()
    buf, w = s.sample_to_host(n, 4, "b8")
    assert bytes(buf[:w]) == want
    with pytest.raises(SymphaseError):
        s.sample_tiled(n, 4)
