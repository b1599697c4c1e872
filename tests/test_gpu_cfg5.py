"""cfg5 (BASELINE.json configs[4]): raw GF(2) product on random M_sym with a
supplied seeded S — bit-exact against the CPU oracle, CSR vs dense variants."""
import numpy as np
import pytest

from paper_2311_03906_b200 import circuits as CI
from paper_2311_03906_b200.sampler import pack_bits

pytestmark = pytest.mark.gpu


def host(t):
    return t.cpu().numpy().view(np.uint64)


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


@pytest.mark.parametrize("dens", CI.CFG5_DENSITIES)
def test_cfg5_shape_product_equals_oracle(gpu_sampler_factory, port, dens):
    """m=1000 x v=10^4 at the cfg5 densities, N=2^14 + 37 (ragged tail)."""
    model = CI.random_msym_model(1000, 10**4, dens, 1e-3, seed=7)
    n = (1 << 14) + 37
    rng = np.random.default_rng(42)
    S = pack_bits(rng.integers(0, 2, size=(model.n_sym, n), dtype=np.uint8))
    want = port.sample(model.row_ptr, model.sym_idx, S, n)
    s = gpu_sampler_factory()
    s.load_csr(model.row_ptr, model.sym_idx, model.n_sym)
    for variant in ("sparse", "dense"):
        s.set_product(variant)
        got = host(s.sample_given(dev(S), n))
        assert np.array_equal(got, want), (dens, variant)


@pytest.mark.parametrize("dens", [0.001, 0.01])
def test_cfg5_full_size_csr_equals_dense(gpu_sampler_factory, port, dens):
    """Full cfg5 shape (10^4 x 10^5, N = 2^20): the CSR and dense products
    agree bit for bit, and a 4096-shot slice matches the oracle."""
    import torch
    model = CI.random_msym_model(10**4, 10**5, dens, 1e-3, seed=7)
    n = 1 << 20
    g = torch.Generator(device="cuda").manual_seed(42)
    S = torch.randint(-(2**63), 2**63 - 1, (model.n_sym, n // 64), dtype=torch.int64,
                      device="cuda", generator=g)
    s = gpu_sampler_factory()
    s.load_csr(model.row_ptr, model.sym_idx, model.n_sym)
    s.set_product("sparse")
    a = s.sample_given(S, n)
    s.set_product("dense")
    b = s.sample_given(S, n)
    assert torch.equal(a, b)
    sl = host(S[:, :64].contiguous())
    want = port.sample(model.row_ptr, model.sym_idx, sl, 4096)
    assert np.array_equal(host(a[:, :64].contiguous()), want)
    del S, a, b
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dens", [0.0005, 0.002])
def test_fused_many_rows_single_buffer(gpu_sampler_factory, port, dens):
    """8000 rows do not fit two shot tiles on chip: the fused sampler runs
    single-buffered, and its records still equal M_sym . S for the S its
    streams draw (and the oracle)."""
    model = CI.random_msym_model(8000, 20000, dens, 2e-3, seed=11)
    s = gpu_sampler_factory(model)
    T = s.shot_tile
    for n in (T, 5 * T + 9):
        out = s.sample(n, 3)
        S = s.draw_assignments(n, 3)
        assert np.array_equal(host(out), host(s.sample_given(S, n)))
    n = 2 * T
    S = s.draw_assignments(n, 4)
    assert np.array_equal(host(s.sample(n, 4)),
                          port.sample(model.row_ptr, model.sym_idx, host(S), n))


def test_sample_without_onchip_tile_uses_draw_and_product(gpu_sampler_factory, port):
    """A model with too many rows for any on-chip tile still samples through
    sp_sample (draw S + explicit product), with counts and host records."""
    import torch
    model = CI.random_msym_model(40000, 3000, 0.002, 0.01, seed=5)
    s = gpu_sampler_factory(model)
    assert not s.plan_info()["fused_ok"]
    n = 3 * 4096 + 77
    counts = torch.zeros(model.n_meas, dtype=torch.int64, device="cuda")
    out = s.sample(n, 9, counts=counts)
    S = s.draw_assignments(n, 9)
    want = port.sample(model.row_ptr, model.sym_idx, host(S), n)
    assert np.array_equal(host(out), want)
    pc = np.unpackbits(want.view(np.uint8), axis=1).sum(axis=1)
    assert np.array_equal(counts.cpu().numpy(), pc)
    buf, w = s.sample_to_host(n, 9, "b8")
    assert bytes(buf[:w]) == port.encode(want, model.n_meas, n, "b8")


def test_many_flips_per_shot_skips_fused_plan(gpu_sampler_factory, port):
    """Dense M_sym with frequent faults (~9e4 bit flips per shot): the planner
    does not build the fused kernel's tables (SP_FUSED_MAX_FLIPS); sp_sample
    draws S and runs the explicit-S product (here the Four-Russians dense
    variant, density 0.5) with the same records as the oracle on that S."""
    model = CI.random_msym_model(300, 2000, 0.5, 0.3, seed=3)
    s = gpu_sampler_factory(model)
    assert not s.plan_info()["fused_ok"]
    n = 5000
    out = s.sample(n, 21)
    S = s.draw_assignments(n, 21)
    assert np.array_equal(host(out), port.sample(model.row_ptr, model.sym_idx, host(S), n))
