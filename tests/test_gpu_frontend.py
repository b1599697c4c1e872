"""The symbolic pass with its phase matrix on the device (frontend_dev.cu,
SP_FRONTEND_DEV=1) gives the same InitResult as the host pass (and so as the
reference, tests/test_frontend_cpu.py) on random, syndrome and Fig. 3
circuits."""
import numpy as np
import pytest

from paper_2311_03906_b200 import circuits as CI
from paper_2311_03906_b200 import run_initialization

pytestmark = pytest.mark.gpu


def both(text, monkeypatch):
    monkeypatch.setenv("SP_FRONTEND_DEV", "0")
    a = run_initialization(text)
    monkeypatch.setenv("SP_FRONTEND_DEV", "1")
    b = run_initialization(text)
    return a, b


def same(a, b):
    return (a.n_sym == b.n_sym and np.array_equal(a.row_ptr, b.row_ptr)
            and np.array_equal(a.sym_idx, b.sym_idx) and a.groups.tobytes() == b.groups.tobytes())


def test_device_phase_store_random_circuits(monkeypatch):
    rng = CI.MT19937_64(77)
    for _ in range(60):
        text = CI.random_test_circuit(rng, n_qubits=1 + rng.below(9), n_instr=5 + rng.below(120))
        a, b = both(text, monkeypatch)
        assert same(a, b), text


@pytest.mark.parametrize("which", ["surface5", "rep", "fig3a", "fig3b", "fig3c", "padded"])
def test_device_phase_store_structured(monkeypatch, which):
    text = {"surface5": lambda: CI.surface_code(5, 5, 1e-3),
            "rep": lambda: CI.repetition_code(5, 5, 0.01),
            "fig3a": lambda: CI.bench_family("a", 120, 1),
            "fig3b": lambda: CI.bench_family("b", 120, 2),
            "fig3c": lambda: CI.bench_family("c", 150, 3),
            "padded": lambda: CI.gate_padding_pair()[1]}[which]()
    a, b = both(text, monkeypatch)
    assert same(a, b)


@pytest.mark.parametrize("which", ["fig3c_300", "fig3b_400", "surface9"])
def test_phase_store_moves_to_device_mid_pass(monkeypatch, which):
    """Default mode: the pass starts on the host and moves its phase matrix
    to the device once measurements XOR > 2^17 words each (fig3c n=300 after
    a few layers); surface codes stay on the host. Same InitResult either way."""
    text = {"fig3c_300": lambda: CI.bench_family("c", 300, 4),
            "fig3b_400": lambda: CI.bench_family("b", 400, 5),
            "surface9": lambda: CI.surface_code(9, 9, 1e-3)}[which]()
    monkeypatch.setenv("SP_FRONTEND_DEV", "0")
    a = run_initialization(text)
    monkeypatch.delenv("SP_FRONTEND_DEV")
    b = run_initialization(text)
    assert same(a, b)
