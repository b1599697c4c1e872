"""K6: the dense explicit-S product as an int8 GEMM on the tensor cores
(tcgen05.mma kind::i8, counts in TMEM, parity) — bit-exact against the CPU
oracle and the other product variants (bit_matrix.cpp:287-312)."""
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


@pytest.mark.parametrize("m,v,n,dens", [(1, 1, 1, 0.5), (5, 40, 70, 0.3), (128, 128, 256, 0.5),
                                        (128, 256, 256, 0.5), (256, 128, 256, 0.5), (128, 128, 512, 0.5),
                                        (128, 131, 256, 0.5), (128, 128, 257, 0.5), (513, 300, 129, 0.5),
                                        (129, 131, 257, 0.5), (300, 1000, 1000, 0.1),
                                        (200, 300, 4096 + 33, 0.9), (1000, 2000, 300, 0.5)])
def test_tensor_product_equals_oracle(gpu_sampler_factory, port, m, v, n, dens):
    """Tile-edge and ragged shapes: rows, symbols and shots on and off the
    128-row / 512-row-CTA / 128-symbol / 128-shot tiles."""
    model = CI.random_msym_model(m, v, dens, 1e-3, seed=m + v)
    rng = np.random.default_rng(n)
    S = pack_bits(rng.integers(0, 2, size=(model.n_sym, n), dtype=np.uint8))
    want = port.sample(model.row_ptr, model.sym_idx, S, n)
    s = gpu_sampler_factory()
    s.load_csr(model.row_ptr, model.sym_idx, model.n_sym)
    s.set_product("tensor")
    got = host(s.sample_given(dev(S), n))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dens", CI.CFG5_DENSITIES)
def test_tensor_product_cfg5_shape(gpu_sampler_factory, port, dens):
    """cfg5 rows/symbols at N = 2^14 + 37: tensor == oracle == Four-Russians."""
    model = CI.random_msym_model(1000, 10**4, dens, 1e-3, seed=7)
    n = (1 << 14) + 37
    rng = np.random.default_rng(42)
    S = pack_bits(rng.integers(0, 2, size=(model.n_sym, n), dtype=np.uint8))
    want = port.sample(model.row_ptr, model.sym_idx, S, n)
    s = gpu_sampler_factory()
    s.load_csr(model.row_ptr, model.sym_idx, model.n_sym)
    s.set_product("tensor")
    assert np.array_equal(host(s.sample_given(dev(S), n)), want)
    s.set_product("dense")
    assert np.array_equal(host(s.sample_given(dev(S), n)), want)


def test_auto_picks_tensor_and_rebuilds_on_reload(gpu_sampler_factory, port):
    """AUTO routes a dense product with >= 4096 symbols to K6; loading another
    model of the same shape must rebuild the u8 operand layout (the buffer is
    reused, so a stale layout would still have the right size)."""
    n = 3 * 4096 + 5
    rng = np.random.default_rng(3)
    s = gpu_sampler_factory()
    for seed in (11, 12):
        model = CI.random_msym_model(700, 5000, 0.5, 1e-3, seed=seed)
        S = pack_bits(rng.integers(0, 2, size=(model.n_sym, n), dtype=np.uint8))
        s.load_csr(model.row_ptr, model.sym_idx, model.n_sym)
        before = s.launches
        got = host(s.sample_given(dev(S), n))
        assert np.array_equal(got, port.sample(model.row_ptr, model.sym_idx, S, n))
        assert s.launches - before == 2  # operand layout + K6
        s.sample_given(dev(S), n)
        assert s.launches - before == 3
