"""Bit-exact parity of the CUDA path (through the C ABI) against the CPU
oracle and the reference's own outputs (tests/golden)."""
import numpy as np
import pytest

from conftest import golden_circuit
from paper_2311_03906_b200 import circuits as CI
from paper_2311_03906_b200 import run_initialization
from paper_2311_03906_b200.sampler import pack_bits

pytestmark = pytest.mark.gpu


def host(t):
    return t.cpu().numpy().view(np.uint64)


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


CASES = ["worked.700.42", "mixed.200.9", "degen.500.99", "dep.1000.42", "rep5.777.1",
         "surf3.1500.2024", "rand3.64.7", "rand5.513.5"]


def test_philox_known_answers(gpu_sampler_factory):
    # Random123 known-answer vectors for philox4x32-10.
    s = gpu_sampler_factory()
    assert s.debug_philox([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    f = 0xFFFFFFFF
    assert s.debug_philox([f, f, f, f], [f, f]) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]


@pytest.mark.parametrize("case", CASES)
def test_compat_draw_equals_reference_draw_assignments(gpu_sampler_factory, golden, case):
    name, n, seed = case.split(".")
    _, init = golden_circuit(golden, name)
    s = gpu_sampler_factory(init, rng="compat")
    S = s.draw_assignments(int(n), int(seed))
    assert np.array_equal(host(S), golden["draws"][case])


@pytest.mark.parametrize("case", CASES + ["det_m0.3.0"])
@pytest.mark.parametrize("fmt", ["01", "b8"])
def test_compat_end_to_end_equals_cliffsym_sample(gpu_sampler_factory, golden, case, fmt):
    """Fused compat kernel + device encode == `cliffsym sample --seed S --format F`."""
    name, n, seed = case.split(".")
    n, seed = int(n), int(seed)
    text, _ = golden_circuit(golden, name)
    init = run_initialization(text)  # our own front end, then our own kernels
    s = gpu_sampler_factory(init, rng="compat")
    m = s.sample(n, seed)
    got = s.encode(m, n, fmt).cpu().numpy().tobytes()
    assert got == golden["cmd_sample"][f"{case}.{fmt}"].tobytes()
    buf, w = s.sample_to_host(n, seed, fmt)
    assert bytes(buf[:w]) == got


def test_compat_fused_equals_oracle_large(gpu_sampler_factory, port):
    init = run_initialization(CI.surface_code(5, 5, 1e-3))
    s = gpu_sampler_factory(init, rng="compat")
    n, seed = 50_000, 7
    got = host(s.sample(n, seed))
    S = port.draw_assignments(init, n, seed)
    assert np.array_equal(host(s.draw_assignments(n, seed)), S)
    assert np.array_equal(got, port.sample(init.row_ptr, init.sym_idx, S, n))


@pytest.mark.parametrize("variant", ["sparse", "dense"])
def test_product_on_supplied_batches_equals_reference(gpu_sampler_factory, golden, variant):
    """K2 == reference sample(expressions, batch) on acceptance-C6-shaped inputs."""
    g = golden["given_s"]
    s = gpu_sampler_factory()
    for i in range(int(g["count"][0])):
        n = int(g[f"{i}.n"][0])
        S = g[f"{i}.S"]
        s.load_csr(g[f"{i}.row_ptr"], g[f"{i}.sym_idx"], S.shape[0])
        s.set_product(variant)
        out = s.sample_given(dev(S), n)
        assert np.array_equal(host(out), g[f"{i}.out"]), (variant, i)


@pytest.mark.parametrize("variant", ["sparse", "dense", "auto"])
def test_product_random_vs_oracle(gpu_sampler_factory, port, variant):
    """K2 on random M_sym / S vs the oracle: CSR walk, Four-Russians dense
    product, and the density-based automatic choice (dense above ~0.17)."""
    rng = np.random.default_rng(5)
    s = gpu_sampler_factory()
    for n_m, n_s, n, dens in [(300, 500, 2048, 0.05), (1000, 3000, 100_000, 0.01),
                              (64, 2000, 70_001, 0.5), (1, 1, 1, 1.0)]:
        bits = (rng.random((n_m, n_s)) < dens).astype(np.uint8)
        rows = [np.nonzero(r)[0].astype(np.uint32) for r in bits]
        rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.uint64)
        si = np.concatenate(rows).astype(np.uint32)
        S = pack_bits(rng.integers(0, 2, size=(n_s, n), dtype=np.uint8))
        s.load_csr(rp, si, n_s)
        s.set_product(variant)
        got = host(s.sample_given(dev(S), n))
        assert np.array_equal(got, port.sample(rp, si, S, n)), (n_m, n_s, n)


def test_product_out_of_range_symbol(gpu_sampler_factory):
    # test_sampler.cpp:114-118
    s = gpu_sampler_factory()
    s.load_csr(np.array([0, 1], np.uint64), np.array([5], np.uint32), 6)
    S = dev(np.zeros((3, 1), np.uint64))
    with pytest.raises(IndexError):
        s.sample_given(S, 8, n_sym_S=3)


@pytest.mark.parametrize("cfg", ["rep", "surf5", "mixed", "thin"])
def test_philox_fused_equals_product_of_its_draws(gpu_sampler_factory, port, cfg):
    """K1 output == M_sym . S for the S its streams draw (bit-exact), and K2(S) == oracle.
    "thin": channels whose non-null patterns all flip one list (DEPOLARIZE1 before a Z
    measurement, DEPOLARIZE2 with one qubit never measured) fire as thinned Bernoulli
    variables in K1; the draw kernel maps each firing back to a pattern and draws the
    null patterns in its second pass, so the identity still holds bit for bit."""
    text = {"rep": CI.repetition_code(5, 5, 0.01), "surf5": CI.surface_code(5, 5, 1e-3),
            "mixed": "H 0\nCX 0 1\nDEPOLARIZE1(0.2) 0\nX_ERROR(0.3) 1\nX_ERROR(1) 1\n"
                     "X_ERROR(0.5) 0\nM 0\nR 1\nH 1\nDEPOLARIZE2(0.7) 0 1\nM 1 0\n",
            "thin": "DEPOLARIZE1(0.3) 0 1 2\nDEPOLARIZE2(0.2) 3 4\nCX 0 3\n"
                    "DEPOLARIZE1(0.01) 3 5\nDEPOLARIZE2(0.05) 5 6\nM 0 1 2 3 5\n"}[cfg]
    init = run_initialization(text)
    s = gpu_sampler_factory(init)
    T = s.shot_tile
    for n in (1, 63, T, 3 * T + 17, 200_000):
        for seed in (0, 42):
            out = s.sample(n, seed)
            S = s.draw_assignments(n, seed)
            assert np.array_equal(host(out), host(s.sample_given(S, n))), (n, seed)
    n = 3 * T + 5
    S = s.draw_assignments(n, 9)
    assert np.array_equal(host(s.sample_given(S, n)),
                          port.sample(init.row_ptr, init.sym_idx, host(S), n))


def test_philox_shot_range_split_is_invariant(gpu_sampler_factory):
    """Any split at shot-tile boundaries (one GPU or many) yields the same bits."""
    init = run_initialization(CI.surface_code(5, 5, 1e-3))
    s = gpu_sampler_factory(init)
    T = s.shot_tile
    n = 8 * T
    whole = host(s.sample(n, 123))
    parts = [host(s.sample(2 * T, 123, shot_begin=b)) for b in range(0, n, 2 * T)]
    assert np.array_equal(whole, np.concatenate(parts, axis=1))
    Sw = host(s.draw_assignments(n, 123))
    Sp = [host(s.draw_assignments(4 * T, 123, shot_begin=b)) for b in (0, 4 * T)]
    assert np.array_equal(Sw, np.concatenate(Sp, axis=1))
    with pytest.raises(ValueError):
        s.sample(T, 1, shot_begin=T // 2)


def test_counts_equal_popcount(gpu_sampler_factory):
    import torch
    init = run_initialization(CI.surface_code(5, 5, 1e-3))
    s = gpu_sampler_factory(init)
    n = 123_457
    counts = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
    out = host(s.sample(n, 5, counts=counts))
    pc = np.unpackbits(out.view(np.uint8), axis=1).sum(axis=1)
    assert np.array_equal(pc, counts.cpu().numpy())


@pytest.mark.parametrize("fmt", ["01", "b8"])
def test_encode_vs_oracle(gpu_sampler_factory, port, fmt):
    rng = np.random.default_rng(11)
    s = gpu_sampler_factory()
    for n_m, n in [(3, 1), (9, 1), (145, 1000), (40, 4097), (1000, 333), (3585, 96)]:
        m = pack_bits(rng.integers(0, 2, size=(n_m, n), dtype=np.uint8))
        got = s.encode(dev(m), n, fmt).cpu().numpy().tobytes()
        assert got == port.encode(m, n_m, n, fmt), (n_m, n)


def test_encode_golden_vectors(gpu_sampler_factory):
    # test_sampler.cpp:120-147
    s = gpu_sampler_factory()
    m = dev(np.array([[1], [0], [1]], dtype=np.uint64))
    assert s.encode(m, 1, "01").cpu().numpy().tobytes() == b"101\n"
    assert s.encode(m, 1, "b8").cpu().numpy().tobytes() == bytes([5])
    nine = dev(np.ones((9, 1), dtype=np.uint64))
    assert s.encode(nine, 1, "b8").cpu().numpy().tobytes() == bytes([0xFF, 1])


def test_sample_zero_shots_rejected(gpu_sampler_factory):
    init = run_initialization("H 0\nM 0\n")
    s = gpu_sampler_factory(init)
    with pytest.raises(ValueError):
        s.sample(0, 1)
    with pytest.raises(ValueError):
        s.draw_assignments(0, 1)


def test_degenerate_and_constant_rows(gpu_sampler_factory):
    # test_sampler.cpp:36-60 under the Philox sampler.
    init = run_initialization("X_ERROR(1) 0\nX_ERROR(0) 1\nM 0 1\nX 2\nM 2 2\n")
    s = gpu_sampler_factory(init)
    bits = np.unpackbits(host(s.sample(500, 99)).view(np.uint8), axis=1, bitorder="little")[:, :500]
    assert bits[0].all() and not bits[1].any() and bits[2].all() and bits[3].all()
    S = np.unpackbits(host(s.draw_assignments(300, 5)).view(np.uint8), axis=1,
                      bitorder="little")[:, :300]
    assert S[0].all() and S[1].all() and not S[2].any()


def test_bench_configs_parity_small(gpu_sampler_factory):
    """cfg2 at reduced N against the oracle through the explicit path."""
    import torch
    init = run_initialization(CI.surface_code(5, 5, 1e-3))
    s = gpu_sampler_factory(init)
    n = 1 << 16
    S = s.draw_assignments(n, 42)
    from oracle import Port
    want = Port().sample(init.row_ptr, init.sym_idx, host(S), n)
    assert np.array_equal(host(s.sample(n, 42)), want)
    torch.cuda.synchronize()


@pytest.mark.parametrize("cfg", ["rep", "surf5", "surf9"])
def test_tiled_layout_equals_measurement_major(gpu_sampler_factory, cfg):
    import torch
    text = {"rep": CI.repetition_code(5, 5, 0.01), "surf5": CI.surface_code(5, 5, 1e-3),
            "surf9": CI.surface_code(9, 9, 1e-3)}[cfg]
    init = run_initialization(text)
    s = gpu_sampler_factory(init)
    T = s.shot_tile
    for n in (1, T + 77, 5 * T):
        c1 = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
        c2 = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
        mm = s.sample(n, 17, counts=c1)
        tl = s.sample_tiled(n, 17, counts=c2)
        assert torch.equal(s.untile(tl, n), mm)
        assert torch.equal(c1, c2)
        for fmt in ("b8", "01"):
            assert torch.equal(s.encode_tiled(tl, n, fmt), s.encode(mm, n, fmt))


@pytest.mark.parametrize("env", [{"SP_GEN_WARPS": "9"}, {"SP_GEN_WARPS": "14"},
                                 {"SP_PAD_PRED": "1"}, {"SP_PAD_PRED": "0"},
                                 {"SP_AUTOTUNE": "0"}, {"SP_ROWSTAGED": "0"}])
def test_launch_shape_does_not_change_records(gpu_sampler_factory, monkeypatch, env):
    """Random streams are keyed by (slice, global tile) only: the warp split,
    padded-XOR mode, autotune and staging choices change speed, not bits."""
    import torch
    for name, text in [("surf5", CI.surface_code(5, 5, 1e-3)), ("surf9", CI.surface_code(9, 3, 1e-3))]:
        init = run_initialization(text)
        base = gpu_sampler_factory(init)
        n = 5 * base.shot_tile + 11
        c0 = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
        want = base.sample(n, 77, counts=c0)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s = gpu_sampler_factory(init)
        c1 = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
        assert torch.equal(s.sample(n, 77, counts=c1), want), (name, env, s.plan_info())
        assert torch.equal(c0, c1)
        for k in env:
            monkeypatch.delenv(k)


def test_reload_same_and_other_model(gpu_sampler_factory, port):
    """Re-loading an identical model keeps the plan and the records; loading
    a different one rebuilds it (checked against the oracle)."""
    a = run_initialization(CI.surface_code(5, 5, 1e-3))
    b = run_initialization(CI.repetition_code(5, 5, 0.01))
    s = gpu_sampler_factory(a)
    n = 3 * s.shot_tile
    first = host(s.sample(n, 5))
    s.load(a)
    assert np.array_equal(host(s.sample(n, 5)), first)
    s.load(b)
    nb = 3 * s.shot_tile
    S = s.draw_assignments(nb, 5)
    assert np.array_equal(host(s.sample(nb, 5)), port.sample(b.row_ptr, b.sym_idx, host(S), nb))
    s.load(a)
    assert np.array_equal(host(s.sample(n, 5)), first)


def test_tile_straddling_shot_counts(gpu_sampler_factory, port):
    """Shot counts around word, tile and the reference's 512-shot tile sizes
    (test_bit_matrix.cpp:328-349 uses 511/512/513/1024/1537): the compat
    sampler equals the oracle's draw_assignments + sample, and the Philox
    sampler equals the product of its own draws."""
    init = run_initialization(CI.surface_code(3, 3, 0.02))
    s = gpu_sampler_factory(init, rng="compat")
    T = s.shot_tile
    ns = sorted({1, 31, 32, 33, 63, 64, 65, 127, 128, 129, 511, 512, 513, 1024, 1537,
                 T - 1, T, T + 1, 2 * T + 3})
    for n in ns:
        got = host(s.sample(n, 17))
        S = port.draw_assignments(init, n, 17)
        assert np.array_equal(got, port.sample(init.row_ptr, init.sym_idx, S, n)), n
    s.set_rng("philox")
    for n in ns:
        out = s.sample(n, 17)
        assert np.array_equal(host(out), host(s.sample_given(s.draw_assignments(n, 17), n))), n


def test_no_measurements(gpu_sampler_factory):
    """A circuit without measurements: empty records, '01' gives one empty
    line per shot and 'b8' nothing (encode_shots, sampler.cpp:118-140)."""
    init = run_initialization("H 0\nCX 0 1\nDEPOLARIZE1(0.1) 0\n")
    assert init.n_meas == 0
    s = gpu_sampler_factory(init)
    out = s.sample(100, 1)
    assert out.shape[0] == 0
    assert s.encode(out, 100, "01", n_meas=0).cpu().numpy().tobytes() == b"\n" * 100
    assert s.encode(out, 100, "b8", n_meas=0).numel() == 0
    buf, w = s.sample_to_host(100, 1, "01")
    assert bytes(buf[:w]) == b"\n" * 100


def test_product_long_rows_split(gpu_sampler_factory, port, monkeypatch):
    """K2 CSR with a few very long rows (a scrambled circuit's final
    measurements can hold 10^5 symbols): the rows are cut into segments
    combined with atomics, and the product still equals the oracle."""
    monkeypatch.setenv("SP_K2_SEG", "64")
    rng = np.random.default_rng(17)
    n_m, n_s, n = 200, 3000, 5000 + 13
    rows = []
    for k in range(n_m):
        length = int(rng.integers(2000, 3000)) if k % 37 == 5 else int(rng.integers(0, 20))
        rows.append(np.sort(rng.choice(n_s, size=length, replace=False)).astype(np.uint32))
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.uint64)
    si = np.concatenate(rows).astype(np.uint32)
    S = pack_bits(rng.integers(0, 2, size=(n_s, n), dtype=np.uint8))
    s = gpu_sampler_factory()
    s.load_csr(rp, si, n_s)
    s.set_product("sparse")
    got = host(s.sample_given(dev(S), n))
    assert np.array_equal(got, port.sample(rp, si, S, n))
