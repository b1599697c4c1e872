"""Detector layer: D_sym = A . M_sym built by
sp_detector_rows, checked with the CPU oracle on supplied S."""
import numpy as np
import pytest

from paper_2311_03906_b200 import circuits as CI
from paper_2311_03906_b200 import run_initialization
from paper_2311_03906_b200.sampler import pack_bits


def _sym_dist(init):
    dist = np.zeros(init.n_sym, dtype=np.uint8)
    for g in init.groups:
        dist[g["first_symbol"]:g["first_symbol"] + g["arity"]] = g["dist"]
    return dist


@pytest.mark.parametrize("d,r", [(3, 3), (5, 5), (5, 2)])
def test_surface_detectors_are_deterministic_without_faults(d, r):
    """Every detector and the observable are free of coin symbols and of
    the constant s0: noiseless, they are always 0."""
    init = run_initialization(CI.surface_code(d, r, 1e-3))
    dets, obs = CI.surface_code_detectors(d, r)
    L = CI.surface_layout(d)
    assert len(dets) == len(L.zanc) * (r + 1) + len(L.xanc) * (r - 1)
    dist = _sym_dist(init)
    for rows in (dets, obs):
        m = init.detector_model(rows)
        assert m.n_meas == len(rows)
        assert not np.any(dist[m.sym_idx] == 2) and not np.any(m.sym_idx == 0)


def test_detector_rows_are_xor_of_measurement_rows(port):
    """For any S: (A . M) S == A (M S), through the oracle product."""
    init = run_initialization(CI.surface_code(3, 3, 1e-2))
    dets, obs = CI.surface_code_detectors(3, 3)
    dm = init.detector_model(dets + obs)
    n = 777
    rng = np.random.default_rng(3)
    S = pack_bits(rng.integers(0, 2, size=(init.n_sym, n), dtype=np.uint8))
    meas = port.sample(init.row_ptr, init.sym_idx, S, n)
    want = np.stack([np.bitwise_xor.reduce(meas[list(rows)], axis=0) for rows in dets + obs])
    assert np.array_equal(port.sample(dm.row_ptr, dm.sym_idx, S, n), want)


def test_detector_rows_errors():
    init = run_initialization(CI.surface_code(3, 3, 1e-3))
    with pytest.raises(IndexError):
        init.detector_model([[0, init.n_meas]])
    empty = init.detector_model([[], [1, 1]])  # empty set and a self-cancelling pair
    assert empty.nnz == 0 and empty.n_meas == 2
