"""Detector layer on the GPU: detector records and counts sampled by the
fused kernel from D_sym = A . M_sym."""
import numpy as np
import pytest

import oracle
from paper_2311_03906_b200 import circuits as CI
from paper_2311_03906_b200 import run_initialization

pytestmark = pytest.mark.gpu

N = 10_000_000
SIGMA = 5.0


def host(t):
    return t.cpu().numpy().view(np.uint64)


def test_detector_flip_rates_10M(gpu_sampler_factory):
    """Per-detector and observable flip rates within 5 sigma of the analytic
    piling-up value at 10^7 shots (cfg2 circuit)."""
    import torch
    init = run_initialization(CI.surface_code(5, 5, 1e-3))
    dets, obs = CI.surface_code_detectors(5, 5)
    dm = init.detector_model(dets + obs)
    s = gpu_sampler_factory(dm)
    counts = torch.zeros(dm.n_meas, dtype=torch.int64, device="cuda")
    out = s.empty_bits(dm.n_meas, N)
    s.sample(N, 99, out=out, counts=counts)
    got = counts.cpu().numpy()
    want = oracle.flip_rates(dm)
    sd = np.sqrt(want * (1 - want) / N)
    bad = [(k, got[k] / N, want[k]) for k in range(dm.n_meas)
           if abs(got[k] / N - want[k]) > SIGMA * sd[k] + 1e-12]
    assert not bad, bad
    # p = 1e-3 detectors fire at ~1-2 %; the raw (undecoded) observable far more
    assert 0.005 < want[:len(dets)].min() and want[:len(dets)].max() < 0.05


def test_detector_sampler_equals_product_of_its_draws(gpu_sampler_factory, port):
    init = run_initialization(CI.surface_code(5, 3, 1e-2))
    dets, obs = CI.surface_code_detectors(5, 3)
    dm = init.detector_model(dets + obs)
    s = gpu_sampler_factory(dm)
    T = s.shot_tile
    for n in (T, 3 * T + 5):
        out = s.sample(n, 4)
        S = s.draw_assignments(n, 4)
        assert np.array_equal(host(out), host(s.sample_given(S, n)))
        # and A . (M S) through the oracle
        meas = port.sample(init.row_ptr, init.sym_idx, host(S), n)
        want = np.stack([np.bitwise_xor.reduce(meas[r], axis=0) for r in dets + obs])
        assert np.array_equal(host(out), want)
