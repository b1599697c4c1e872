"""Per-detector flip counts in the sampling launch (sp_sample_ex): the fused
kernel's drain counts each detector from the finished rows, so the counts
must equal the popcount of the XOR of the detector's measurement records,
read back from the records the same launch wrote — bit-exact integers.

BASELINE configs[2] (cfg3) all-reduces per-detector counts over the GPUs;
the reference has no DETECTOR instruction (circuit.cpp:117-121), so the
detector sets are the standard memory-Z ones (circuits.surface_code_detectors)
plus irregular ones that exercise the general (non-row) detector path."""
import numpy as np
import pytest

from paper_2311_03906_b200 import circuits as CI
from paper_2311_03906_b200 import run_initialization

pytestmark = pytest.mark.gpu


def host(t):
    return t.cpu().numpy().view(np.uint64)


def popcount_rows(bits):
    b = bits.view(np.uint8)
    return np.unpackbits(b, axis=-1).sum(axis=-1).astype(np.int64)


def expected(meas, dets):
    return np.array([popcount_rows(np.bitwise_xor.reduce(meas[d], axis=0)[None])[0]
                     if len(d) else 0 for d in dets])


def irregular(n_meas, rng):
    """Detectors the row shortcut cannot take: long sets, repeats that
    cancel, duplicates of a row detector, single non-root rows, empty."""
    out = [sorted(rng.choice(n_meas, size=5, replace=False).tolist()) for _ in range(20)]
    out += [[3, 3, 7], [n_meas - 1], [], [0, 0]]
    return out


@pytest.mark.parametrize("d,r,p,tiled", [(5, 5, 1e-2, False), (5, 5, 1e-2, True),
                                          (9, 9, 3e-3, True)])
def test_detector_counts_equal_records(gpu_sampler_factory, d, r, p, tiled):
    import torch
    init = run_initialization(CI.surface_code(d, r, p))
    dets, obs = CI.surface_code_detectors(d, r)
    rng = np.random.default_rng(d * 100 + r)
    all_dets = dets + obs + irregular(init.n_meas, rng) + dets[:3]
    s = gpu_sampler_factory(init)
    s.set_detectors(all_dets)
    T = s.shot_tile
    for n, begin in ((T, 0), (5 * T + 77, 2 * T)):  # a partial last tile too
        cnt = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
        dcnt = torch.zeros(len(all_dets), dtype=torch.int64, device="cuda")
        out = s.sample_counted(n, 31, shot_begin=begin, counts=cnt, det_counts=dcnt, tiled=tiled)
        meas = host(s.untile(out, n) if tiled else out)
        # the records themselves are those of the plain sampler
        plain = s.sample_tiled(n, 31, shot_begin=begin) if tiled else s.sample(n, 31, shot_begin=begin)
        assert np.array_equal(host(out), host(plain))
        assert np.array_equal(cnt.cpu().numpy(), popcount_rows(meas))
        assert np.array_equal(dcnt.cpu().numpy(), expected(meas, all_dets))


def test_detector_counts_cfg3(gpu_sampler_factory):
    """The bench workload: d = 15, 15 rounds, p = 1e-3, tiled records."""
    import torch
    init = run_initialization(CI.surface_code(15, 15, 1e-3))
    dets, obs = CI.surface_code_detectors(15, 15)
    s = gpu_sampler_factory(init)
    s.set_detectors(dets + obs)
    n = 40 * s.shot_tile + 3
    dcnt = torch.zeros(len(dets) + 1, dtype=torch.int64, device="cuda")
    out = s.sample_counted(n, 5, det_counts=dcnt, tiled=True)
    meas = host(s.untile(out, n))
    assert np.array_equal(dcnt.cpu().numpy(), expected(meas, dets + obs))


def test_detector_counts_errors(gpu_sampler_factory):
    import torch
    from paper_2311_03906_b200._native import OutOfRange, SymphaseError
    init = run_initialization(CI.surface_code(3, 3, 1e-2))
    s = gpu_sampler_factory(init)
    dcnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    with pytest.raises(SymphaseError, match="no detectors registered"):
        s.sample_counted(64, 1, det_counts=dcnt)
    with pytest.raises(OutOfRange):
        s.set_detectors([[init.n_meas]])
