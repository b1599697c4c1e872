"""CPU unit tests of the planner's host stages (plan_stages.cpp): chain
transform, drain plan and detector classification, and the exactness of the
DEPOLARIZE mechanism decomposition (enumerated distributions)."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_2311_03906_b200" / "csrc"


def test_plan_stages(tmp_path):
    cxx = shutil.which("g++")
    if cxx is None:
        pytest.skip("no host C++ compiler")
    exe = tmp_path / "test_plan_stages"
    subprocess.run([cxx, "-std=c++20", "-O2", f"-I{CSRC}", str(ROOT / "tests" / "cpp" / "test_plan_stages.cpp"),
                    str(CSRC / "plan_stages.cpp"), "-o", str(exe)], check=True, capture_output=True,
                   text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " 0 failed" in r.stdout
