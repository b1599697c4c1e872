"""The BASELINE headline shapes on the GPU: cfg3 (rotated surface code d=15,
15 rounds: 3,585 measurements, 101,490 symbols; the configuration the bench
reports) and cfg4 (random Clifford n=1000: 1,899 coin rows, 72,723 channels on
one row, merged into one variable by default).

* front end == the reference's run_initialization (tableau.cpp:318-382), via
  the digests in tests/golden/large.json (the phase store may move to the
  device on a GPU box, so this runs here too);
* K1 records == M_sym . S of the S its own streams draw (bit-exact), in both
  record layouts, over >= 4 shot tiles with a ragged tail (sampler.cpp:48-112);
  cfg4 with channel merging off (SP_MERGE_MIN=0), where the identity holds;
* per-measurement (and, at cfg3, per-detector) flip rates within 5 sigma of
  the analytic piling-up value at 10^7 shots, cfg4 with merging on."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2311_03906_b200 import circuits as CI
from paper_2311_03906_b200 import run_initialization

pytestmark = pytest.mark.gpu

N = 10_000_000
SIGMA = 5.0
LARGE = json.loads((Path(__file__).resolve().parent / "golden" / "large.json").read_text())


def host(t):
    return t.cpu().numpy().view(np.uint64)


_INIT = {}


def init_of(cfg):
    if cfg not in _INIT:
        _INIT[cfg] = run_initialization(CI.CONFIGS[cfg]["text"]())
    return _INIT[cfg]


def digest_ok(init, want):
    import hashlib

    def d(a, dt):
        a = np.ascontiguousarray(np.asarray(a).astype(dt))
        return {"len": int(a.size), "dtype": str(a.dtype),
                "sha256": hashlib.sha256(a.tobytes()).hexdigest()}
    g = init.groups
    return (init.n_meas == want["n_meas"] and init.n_sym == want["n_sym"]
            and d(init.row_ptr, np.uint64) == want["row_ptr"]
            and d(init.sym_idx, np.uint32) == want["sym_idx"]
            and d(g["dist"], np.uint8) == want["dist"]
            and d(g["param"], np.float64) == want["param"]
            and d(g["first_symbol"], np.uint32) == want["first"]
            and d(g["arity"], np.uint32) == want["arity"])


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg4"])
def test_front_end_matches_reference_pass_on_gpu_box(cfg):
    assert digest_ok(init_of(cfg), LARGE[cfg])


def _product_identity(s, n, seed, tiled):
    import torch
    if tiled:
        t = torch.empty(s.tiled_words(n), dtype=torch.int64, device="cuda")
        s.sample_tiled(n, seed, out=t)
        got = s.untile(t, n)
    else:
        got = s.sample(n, seed)
    S = s.draw_assignments(n, seed)
    want = s.sample_given(S, n)
    return np.array_equal(host(got), host(want)), S, want


@pytest.mark.parametrize("tiled", [True, False])
def test_cfg3_fused_equals_product_of_its_draws(gpu_sampler_factory, port, tiled):
    init = init_of("cfg3")
    s = gpu_sampler_factory(init)
    info = s.plan_info()
    assert info["fused_ok"] in (1, 3, 4, 5), info  # the fused sampler the bench runs (K1 or its queued form K7)
    T = s.shot_tile
    for n, seed in ((4 * T + 37, 3), (16 * T, 11), (1, 5)):
        ok, S, want = _product_identity(s, n, seed, tiled)
        assert ok, (n, seed)
    n = 4 * T + 37
    ok, S, want = _product_identity(s, n, 21, tiled)
    assert ok
    # ... and the explicit product equals the CPU oracle on that S
    assert np.array_equal(host(want), port.sample(init.row_ptr, init.sym_idx, host(S), n))


def test_cfg3_shot_range_split_is_invariant(gpu_sampler_factory):
    import torch
    s = gpu_sampler_factory(init_of("cfg3"))
    T = s.shot_tile
    n = 8 * T
    whole = host(s.sample(n, 99))
    parts = [host(s.sample(3 * T, 99, shot_begin=0)), host(s.sample(5 * T, 99, shot_begin=3 * T))]
    assert np.array_equal(whole[:, :3 * T // 64], parts[0][:, :3 * T // 64])
    assert np.array_equal(whole[:, 3 * T // 64:], parts[1][:, :5 * T // 64])


def test_cfg4_unmerged_fused_equals_product_of_its_draws(gpu_sampler_factory, port,
                                                          monkeypatch):
    monkeypatch.setenv("SP_MERGE_MIN", "0")
    init = init_of("cfg4")
    s = gpu_sampler_factory(init)
    T = s.shot_tile
    for tiled in (True, False):
        for n, seed in ((4 * T + 37, 4), (3, 8)):
            ok, S, want = _product_identity(s, n, seed, tiled)
            assert ok, (tiled, n, seed)
    n = 2 * T + 9
    ok, S, want = _product_identity(s, n, 13, False)
    assert ok
    assert np.array_equal(host(want), port.sample(init.row_ptr, init.sym_idx, host(S), n))


def _rates_ok(s, init, seed, tiled):
    import torch
    counts = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
    if tiled:
        out = torch.empty(s.tiled_words(N), dtype=torch.int64, device="cuda")
        s.sample_tiled(N, seed, out=out, counts=counts)
    else:
        out = s.empty_bits(init.n_meas, N)
        s.sample(N, seed, out=out, counts=counts)
    del out
    got = counts.cpu().numpy()
    want = oracle.flip_rates(init)
    sd = np.sqrt(np.maximum(want * (1 - want), 1e-300) / N)
    bad = np.nonzero(np.abs(got / N - want) > SIGMA * sd + 1e-12)[0]
    return [(int(k), got[k] / N, want[k], sd[k]) for k in bad[:20]]


def test_cfg3_per_measurement_flip_rates_10M(gpu_sampler_factory):
    init = init_of("cfg3")
    assert not _rates_ok(gpu_sampler_factory(init), init, 123, tiled=True)


def test_cfg3_per_detector_flip_rates_10M(gpu_sampler_factory):
    dets, obs = CI.surface_code_detectors(15, 15)
    init = init_of("cfg3").detector_model(dets + obs)
    assert not _rates_ok(gpu_sampler_factory(init), init, 321, tiled=True)


def test_cfg4_merged_flip_rates_10M(gpu_sampler_factory):
    init = init_of("cfg4")
    s = gpu_sampler_factory(init)
    assert not _rates_ok(s, init, 456, tiled=True)
