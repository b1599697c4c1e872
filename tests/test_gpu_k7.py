"""K7, the queued form of the fused sampler (k7_queued.cuh, SP_QUEUED=1): the
same slices and streams as K1, so records and counts must be bit-identical
for a seed — in both layouts, with ragged tails and detector counts."""
import os

import pytest
import torch

from paper_2311_03906_b200 import Sampler, circuits, run_initialization

pytestmark = pytest.mark.gpu


def _pair(init, monkeypatch, **env):
    monkeypatch.setenv("SP_QUEUED", "0")
    k1 = Sampler(init)
    monkeypatch.setenv("SP_QUEUED", "1")
    for k, v in env.items():
        monkeypatch.setenv(k, str(v))
    k7 = Sampler(init)
    return k1, k7


@pytest.mark.parametrize("cfg,shots", [("cfg1", 100_003), ("cfg2", 300_001), ("cfg3", 40_000),
                                       ("cfg4", 30_001)])
@pytest.mark.parametrize("tiled", [False, True])
def test_queued_equals_fused(cfg, shots, tiled, monkeypatch):
    init = run_initialization(circuits.CONFIGS[cfg]["text"]())
    k1, k7 = _pair(init, monkeypatch)
    outs = []
    for s in (k1, k7):
        counts = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
        if tiled:
            out = torch.zeros(s.tiled_words(shots), dtype=torch.int64, device="cuda")
            s.sample_tiled(shots, 11, out=out, counts=counts)
        else:
            out = s.sample(shots, 11, counts=counts)
        outs.append((out, counts))
    assert int((outs[0][0] != 0).sum()) > 0
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("shape", [(4, 4, 2), (6, 12, 4), (12, 12, 8)])
def test_queued_shapes_and_detector_counts(shape, monkeypatch):
    """Walker / apply warp counts and ring depth are launch parameters only."""
    init = run_initialization(circuits.CONFIGS["cfg2"]["text"]())
    dets, obs = circuits.surface_code_detectors(5, 5)
    k1, k7 = _pair(init, monkeypatch, SP_Q_WALK=shape[0], SP_Q_APPLY=shape[1], SP_Q_DEPTH=shape[2])
    n = 200_000
    res = []
    for s in (k1, k7):
        s.set_detectors(dets + obs)
        dc = torch.zeros(len(dets) + 1, dtype=torch.int64, device="cuda")
        out = torch.zeros(s.tiled_words(n), dtype=torch.int64, device="cuda")
        s.sample_counted(n, 5, out=out, det_counts=dc, tiled=True)
        res.append((out, dc))
    assert torch.equal(res[0][0], res[1][0])
    assert torch.equal(res[0][1], res[1][1])
    assert int(res[0][1].sum()) > 0


def test_queued_falls_back_when_not_eligible(monkeypatch):
    """A plan with DEPOLARIZE pattern walks (mechanisms off) is served by K1."""
    monkeypatch.setenv("SP_MECH", "0")
    init = run_initialization(circuits.CONFIGS["cfg1"]["text"]())
    k1, k7 = _pair(init, monkeypatch)
    a = k1.sample(50_000, 3)
    b = k7.sample(50_000, 3)
    assert torch.equal(a, b)


@pytest.mark.parametrize("cfg,shots", [("cfg2", 200_000), ("cfg3", 20_000)])
@pytest.mark.parametrize("queued", ["0", "1"])
def test_texture_list_fetch_equals_global_loads(cfg, shots, queued, monkeypatch):
    """The flip lists read through the texture pipe (default) or with
    ld.global.nc (SP_LIST_TEX=0; K7 then falls back to K1) give the same records."""
    init = run_initialization(circuits.CONFIGS[cfg]["text"]())
    monkeypatch.setenv("SP_QUEUED", queued)
    outs = []
    for tex in ("1", "0"):
        monkeypatch.setenv("SP_LIST_TEX", tex)
        s = Sampler(init)
        out = torch.zeros(s.tiled_words(shots), dtype=torch.int64, device="cuda")
        s.sample_tiled(shots, 21, out=out)
        outs.append(out)
    assert int((outs[0] != 0).sum()) > 0
    assert torch.equal(outs[0], outs[1])
