import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.Port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.have_ref():
        pytest.skip("reference library (oracle/_ref) not built here")
    return oracle.Ref()


@pytest.fixture(scope="session")
def golden():
    return {name: np.load(GOLDEN / f"{name}.npz")
            for name in ("frontend", "draws", "cmd_sample", "given_s")}


def golden_circuit(g, name):
    """Reconstructs an InitResult from the frontend fixture."""
    from paper_2311_03906_b200.sampler import GROUP_DTYPE, InitResult
    f = g["frontend"]
    groups = np.zeros(len(f[f"{name}.dist"]), dtype=GROUP_DTYPE)
    groups["dist"] = f[f"{name}.dist"]
    groups["param"] = f[f"{name}.param"]
    groups["first_symbol"] = f[f"{name}.first"]
    groups["arity"] = f[f"{name}.arity"]
    text = f[f"{name}.text"].tobytes().decode()
    return text, InitResult(0, int(f[f"{name}.n_sym"][0]), f[f"{name}.row_ptr"],
                            f[f"{name}.sym_idx"], groups)


@pytest.fixture(scope="session")
def gpu_sampler_factory():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2311_03906_b200 import Sampler

    def make(init=None, rng="philox"):
        return Sampler(init, device=0, rng=rng)
    return make
