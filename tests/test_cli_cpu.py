"""CLI mirror of `cliffsym analyze` (CPU-only part) and the M_sym cache."""
import subprocess
import sys
from pathlib import Path

import numpy as np

from paper_2311_03906_b200 import circuits, run_initialization
from paper_2311_03906_b200.sampler import InitResult

ROOT = Path(__file__).resolve().parents[1]


def run_cli(args, stdin=""):
    return subprocess.run([sys.executable, "-m", "paper_2311_03906_b200"] + args, input=stdin,
                          capture_output=True, text=True, cwd=ROOT, timeout=120)


def test_analyze_worked_example():
    # acceptance.cpp:110-138 criterion 1: m1 = s3, m2 = s1 ^ s2 ^ s3
    r = run_cli(["analyze"], "H 0\nCX 0 1\nX_ERROR(0.1) 0 1\nM 0 1\n")
    assert r.returncode == 0
    lines = [l for l in r.stdout.splitlines() if not l.startswith("#")]
    assert lines == ["m1 = s3", "m2 = s1 ^ s2 ^ s3"]


def test_analyze_constant_and_empty():
    r = run_cli(["analyze"], "X 0\nM 0\nM 1\n")
    assert r.stdout.splitlines()[:2] == ["m1 = 1", "m2 = 0"]


def test_parse_error_exit_code():
    # cliffsym.cpp:346-355 / test_cli.cpp:175-184: parse failures exit 1
    r = run_cli(["analyze"], "H 0\nFROB 1\n")
    assert r.returncode == 1 and "line 2" in r.stderr
    assert run_cli(["frobnicate"]).returncode == 1


def test_msym_cache_round_trip(tmp_path):
    init = run_initialization(circuits.surface_code(3, 3, 0.01))
    p = tmp_path / "m.npz"
    init.save(p)
    back = InitResult.load(p)
    assert back.n_sym == init.n_sym and back.n_qubits == init.n_qubits
    assert np.array_equal(back.row_ptr, init.row_ptr)
    assert np.array_equal(back.sym_idx, init.sym_idx)
    assert back.groups.tobytes() == init.groups.tobytes()
