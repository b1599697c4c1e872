"""Acceptance C8 (acceptance.cpp:437-533), second half, on the device: the
cost of a shot does not depend on circuit length. The sampling time of the
C8 circuit and of the same circuit padded with 100,000 gates (self-inverse
pairs, identical M_sym) must agree within 1.25x, as the reference requires
of its CPU sampler (best of 5, draw + sample + b8 encode)."""
import pytest

from paper_2311_03906_b200 import circuits as CI
from paper_2311_03906_b200 import run_initialization

pytestmark = pytest.mark.gpu


def test_sampling_time_independent_of_gate_count(gpu_sampler_factory):
    import torch
    base, padded = CI.gate_padding_pair()
    n = 2_000_000

    def best_ms(text):
        s = gpu_sampler_factory(run_initialization(text))
        out = s.sample(n, 11)
        s.encode(out, n, "b8")
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = s.sample(n, 11, out=out)
            enc = s.encode(out, n, "b8")
            b.record()
            torch.cuda.synchronize()
            assert enc.numel() > 0
            ts.append(a.elapsed_time(b))
        return min(ts)

    tb, tp = best_ms(base), best_ms(padded)
    assert max(tb, tp) / min(tb, tp) <= 1.25, (tb, tp)
