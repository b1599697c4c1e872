"""The reference's own sampler unit tests (test_sampler.cpp), re-hosted on the
C++ shim include/cliffsym_b200.hpp and run against libsymphase_b200.so."""
import shutil
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_reference_sampler_suite_on_shim(tmp_path):
    cxx = shutil.which("g++")
    if cxx is None:
        pytest.skip("no host C++ compiler")
    exe = tmp_path / "test_shim"
    cmd = [cxx, "-std=c++20", "-O2", f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include",
           str(ROOT / "tests" / "cpp" / "test_shim.cpp"), "-o", str(exe),
           f"-L{ROOT / 'paper_2311_03906_b200'}", "-lsymphase_b200", "-L/usr/local/cuda/lib64",
           "-lcudart", f"-Wl,-rpath,{ROOT / 'paper_2311_03906_b200'}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


REF_BIN = ROOT / "oracle" / "_ref"


@pytest.mark.parametrize("name", ["test_sampler_on_shim", "acceptance_c568_on_shim"])
def test_reference_tests_unchanged_on_shim(name):
    """The reference's test_sampler.cpp (whole) and acceptance criteria 5, 6, 8
    compiled unchanged against the shim (oracle/Makefile `shimtests`, built
    where /root/reference exists; the binaries travel with the repo)."""
    exe = REF_BIN / name
    if not exe.exists():
        pytest.skip("built only where the reference sources are present (oracle/Makefile)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    if name == "test_sampler_on_shim":
        assert " 0 failed," in r.stdout and "FAILED" not in r.stdout, r.stdout
    else:
        assert r.stdout.count("[PASS]") == 3, r.stdout
