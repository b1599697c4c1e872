"""Statistical parity of the in-kernel Philox sampler (north star: per-variable
marginals and per-measurement flip rates within 5 sigma at 10^7 shots).

Analytic targets follow fill_group's pmf (sampler.cpp:11-44) and the
piling-up form of test_sampler.cpp:189-203, computed by oracle.flip_rates."""
import numpy as np
import pytest

import oracle
from paper_2311_03906_b200 import circuits as CI
from paper_2311_03906_b200 import run_initialization

pytestmark = pytest.mark.gpu

N = 10_000_000
SIGMA = 5.0


def within(hits, n, p):
    sd = np.sqrt(max(p * (1 - p), 1e-300) / n)
    return abs(hits / n - p) <= SIGMA * sd + 1e-12, (hits / n, p, sd)


def host(t):
    return t.cpu().numpy().view(np.uint64)


CHANNELS = [("X_ERROR", p) for p in (1e-4, 1e-3, 0.01, 0.1, 0.3, 0.5, 0.9, 1.0, 0.0)] + \
           [("DEPOLARIZE1", p) for p in (1e-3, 0.05, 0.3, 0.75, 1.0)] + \
           [("DEPOLARIZE2", p) for p in (1e-3, 0.1, 0.8, 1.0)]


def channel_circuit():
    lines, q = [], 0
    for name, p in CHANNELS:
        if name == "DEPOLARIZE2":
            lines.append(f"{name}({p!r}) {q} {q + 1}")
            q += 2
        else:
            lines.append(f"{name}({p!r}) {q}")
            q += 1
    lines.append("H " + " ".join(str(i) for i in range(q, q + 3)))  # three fair coins
    lines.append("M " + " ".join(str(i) for i in range(q + 3)))
    return "\n".join(lines) + "\n"


def test_per_variable_marginals_10M(gpu_sampler_factory):
    init = run_initialization(channel_circuit())
    s = gpu_sampler_factory(init)
    S = host(s.draw_assignments(N, 2024))
    tail = N % 64
    valid = np.full(S.shape[1], ~np.uint64(0), dtype=np.uint64)
    if tail:
        valid[-1] = np.uint64((1 << tail) - 1)
    pc = lambda w: int(np.bitwise_count(w & valid).sum())  # noqa: E731
    g = init.groups
    bad = []
    for gi in range(1, len(g)):
        d, p, f = int(g["dist"][gi]), float(g["param"][gi]), int(g["first_symbol"][gi])
        if d in (1, 2):
            q = 0.5 if d == 2 else p
            ok, info = within(pc(S[f]), N, q)
            if not ok:
                bad.append((gi, d, info))
        elif d == 3:  # patterns x, z, y each p/3; identity 1-p
            x, z = S[f], S[f + 1]
            for pat, w in ((1, x & ~z), (2, ~x & z), (3, x & z), (0, ~x & ~z)):
                ok, info = within(pc(w), N, (1 - p) if pat == 0 else p / 3)
                if not ok:
                    bad.append((gi, d, pat, info))
        elif d == 4:  # 15 non-identity patterns each p/15
            rows = [S[f + b] for b in range(4)]
            for pat in range(16):
                w = valid.copy()
                for b in range(4):
                    w &= rows[b] if (pat >> b) & 1 else ~rows[b]
                ok, info = within(pc(w), N, (1 - p) if pat == 0 else p / 15)
                if not ok:
                    bad.append((gi, d, pat, info))
    assert not bad, bad


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "xor_conv", "channels"])
def test_per_measurement_flip_rates_10M(gpu_sampler_factory, cfg):
    import torch
    text = {"cfg1": lambda: CI.repetition_code(5, 5, 0.01),
            "cfg2": lambda: CI.surface_code(5, 5, 1e-3),
            # test_sampler.cpp:193-194
            "xor_conv": lambda: "X_ERROR(0.05) 0\nX_ERROR(0.2) 0\nX_ERROR(0.45) 0\nM 0\n",
            "channels": channel_circuit}[cfg]()
    init = run_initialization(text)
    s = gpu_sampler_factory(init)
    counts = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
    out = s.empty_bits(init.n_meas, N)
    s.sample(N, 77, out=out, counts=counts)
    got = counts.cpu().numpy()
    want = oracle.flip_rates(init)
    bad = [(k, *within(int(got[k]), N, float(want[k]))[1]) for k in range(init.n_meas)
           if not within(int(got[k]), N, float(want[k]))[0]]
    assert not bad, bad
    if cfg == "xor_conv":
        assert abs(want[0] - 0.5 * (1 - 0.9 * 0.6 * 0.1)) < 1e-12


def test_thinned_pattern_marginals_10M(gpu_sampler_factory):
    """Thinned channels (abi.cpp: single-list groups fire as Bernoulli(p_eff) in
    K1): the draw kernel's pattern choice and its null-pattern pass keep every
    pattern at p / #patterns — DEPOLARIZE1 measured in Z (Z is null) and
    DEPOLARIZE2 with one qubit never measured (7 of 15 patterns null), at rates
    where null events often coincide with firings and must be dropped."""
    text = "DEPOLARIZE1(0.45) 0\nDEPOLARIZE2(0.6) 1 2\nDEPOLARIZE2(0.01) 3 4\nM 0 1 3\n"
    init = run_initialization(text)
    s = gpu_sampler_factory(init)
    S = host(s.draw_assignments(N, 77))
    g = init.groups
    bad = []
    for gi in range(1, len(g)):
        d, p, f = int(g["dist"][gi]), float(g["param"][gi]), int(g["first_symbol"][gi])
        arity = 2 if d == 3 else 4
        n_pat = (1 << arity) - 1
        rows = [S[f + b] for b in range(arity)]
        for pat in range(n_pat + 1):
            w = np.full(S.shape[1], ~np.uint64(0), dtype=np.uint64)
            for b in range(arity):
                w &= rows[b] if (pat >> b) & 1 else ~rows[b]
            ok, info = within(int(np.bitwise_count(w).sum()), N, (1 - p) if pat == 0 else p / n_pat)
            if not ok:
                bad.append((gi, pat, info))
    assert not bad, bad
    # and the records K1 makes are the product of exactly these draws
    out = s.sample(N, 77)
    assert np.array_equal(host(out), host(s.sample_given(s.draw_assignments(N, 77), N)))


def test_seeds_differ_and_repeat(gpu_sampler_factory):
    init = run_initialization(CI.surface_code(5, 5, 1e-3))
    s = gpu_sampler_factory(init)
    a = host(s.sample(100_000, 1))
    assert np.array_equal(a, host(s.sample(100_000, 1)))
    assert not np.array_equal(a, host(s.sample(100_000, 2)))


@pytest.mark.parametrize("p,expect", [(1e-9, 0.1), (1e-6, 100.0), (1e-4, 10_000.0)])
def test_tiny_rates_no_spurious_firings(gpu_sampler_factory, p, expect):
    """Skips far longer than a segment must not wrap the warp's position scan
    (kernels.cu geo_skip clamps at 2^22): flip totals follow the rate."""
    import torch
    n_q, shots = 100, 1_000_000
    text = f"X_ERROR({p!r}) " + " ".join(map(str, range(n_q))) + "\nM " + \
        " ".join(map(str, range(n_q))) + "\n"
    init = run_initialization(text)
    s = gpu_sampler_factory(init)
    counts = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
    s.sample(shots, 3, counts=counts)
    total = int(counts.sum().item())
    assert abs(total - expect) <= 5 * max(expect, 1.0) ** 0.5 + 3, (p, total, expect)


def test_merged_channels_rates_10M(gpu_sampler_factory):
    """Channels whose only effect is the same flip list merge into one
    Bernoulli with the piling-up rate (abi.cpp, channel merging): the record
    rates still match the analytic values, draw_assignments still draws every
    original symbol, and SP_MERGE_MIN=0 (no merging) agrees in distribution."""
    import os
    import torch
    text = "X_ERROR(0.001) 0\n" * 300 + "DEPOLARIZE1(0.002) 1\n" * 200 + \
           "CX 0 2\nX_ERROR(0.01) 2\nM 0 1 2\n"
    init = run_initialization(text)
    want = oracle.flip_rates(init)
    for env in ("64", "0"):
        os.environ["SP_MERGE_MIN"] = env
        try:
            s = gpu_sampler_factory(init)
            counts = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
            s.sample(N, 31, counts=counts)
            got = counts.cpu().numpy()
            for k in range(init.n_meas):
                ok, detail = within(int(got[k]), N, float(want[k]))
                assert ok, (env, k, detail)
            S = host(s.draw_assignments(4096, 5))
            assert S.shape[0] == init.n_sym
        finally:
            del os.environ["SP_MERGE_MIN"]


def test_coin_words_independent(gpu_sampler_factory):
    """Fair coins (64 H-then-M qubits; Philox words per (symbol, 128-shot quad)) at 2^22 shots:
    every coin, the agreement of neighbouring coins, of consecutive shots and
    of shots across 128-shot quad boundaries are all 1/2 within 5 sigma."""
    n_q, n = 64, 1 << 22
    text = "H " + " ".join(map(str, range(n_q))) + "\nM " + " ".join(map(str, range(n_q))) + "\n"
    init = run_initialization(text)
    s = gpu_sampler_factory(init)
    rec = host(s.sample(n, 2025))
    bits = np.unpackbits(rec.view(np.uint8), axis=1, bitorder="little")[:, :n].astype(np.int8)

    def half(hits, trials):
        sd = np.sqrt(0.25 / trials)
        return abs(hits / trials - 0.5) <= SIGMA * sd

    assert all(half(int(bits[k].sum()), n) for k in range(n_q))
    assert all(half(int((bits[k] == bits[k + 1]).sum()), n) for k in range(n_q - 1))
    assert all(half(int((bits[k, :-1] == bits[k, 1:]).sum()), n - 1) for k in range(n_q))
    b = bits[:, 127::128][:, :-1] == bits[:, 128::128]
    assert half(int(b.sum()), b.size)
