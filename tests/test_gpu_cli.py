"""`python -m paper_2311_03906_b200 sample` against `cliffsym sample` outputs
(tests/golden/cmd_sample.npz) and the test_cli.cpp contract."""
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import golden_circuit

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def run_cli(args, stdin=""):
    return subprocess.run([sys.executable, "-m", "paper_2311_03906_b200"] + args,
                          input=stdin.encode(), capture_output=True, cwd=ROOT, timeout=300)


@pytest.mark.parametrize("fmt", ["01", "b8"])
def test_sample_compat_is_byte_identical_to_cliffsym(golden, fmt, tmp_path):
    text, _ = golden_circuit(golden, "worked")
    inp = tmp_path / "c.stim"
    inp.write_text(text)
    r = run_cli(["sample", "--in", str(inp), "--shots", "700", "--seed", "42", "--format", fmt,
                 "--rng", "compat"])
    assert r.returncode == 0, r.stderr
    assert r.stdout == golden["cmd_sample"][f"worked.700.42.{fmt}"].tobytes()
    assert b"init_seconds=" in r.stderr and b"sampling_seconds=" in r.stderr


def test_deterministic_circuit_constant_lines():
    # test_cli.cpp:117-122
    r = run_cli(["sample", "--shots", "3"], "M 0\n")
    assert r.returncode == 0 and r.stdout == b"0\n0\n0\n"


def test_reproducible_and_shots_zero_rejected():
    a = run_cli(["sample", "--shots", "500", "--seed", "42", "--format", "b8"], "H 0\nM 0\n")
    b = run_cli(["sample", "--shots", "500", "--seed", "42", "--format", "b8"], "H 0\nM 0\n")
    assert a.returncode == 0 and a.stdout == b.stdout and len(a.stdout) == 500
    assert run_cli(["sample", "--shots", "0"], "M 0\n").returncode == 1


def test_analyze_on_dumped_assignments_matches_sample(tmp_path):
    # test_cli.cpp:124-163
    text = ("H 0\nCX 0 1\nDEPOLARIZE1(0.2) 0\nX_ERROR(0.3) 1\n"
            "M 0\nR 1\nH 1\nM 1 0\n")
    inp = tmp_path / "m.stim"
    inp.write_text(text)
    dump, shots = tmp_path / "a.txt", tmp_path / "s.txt"
    for rng in ("philox", "compat"):
        r = run_cli(["sample", "--in", str(inp), "--shots", "200", "--seed", "9", "--out",
                     str(shots), "--dump-assignments", str(dump), "--rng", rng])
        assert r.returncode == 0, r.stderr
        a = run_cli(["analyze", "--in", str(inp)])
        exprs = []
        for line in a.stdout.decode().splitlines():
            if line.startswith("#"):
                continue
            rhs = line.split(" = ")[1]
            exprs.append([] if rhs == "0" else [0 if t == "1" else int(t[1:])
                                                for t in rhs.split(" ^ ")])
        rows = dump.read_text().splitlines()
        for j, shot_line in enumerate(shots.read_text().splitlines()):
            for k, e in enumerate(exprs):
                v = sum(rows[s][j] == "1" for s in e) % 2
                assert str(v) == shot_line[k], (rng, j, k)


def test_sample_detectors_file(tmp_path):
    """--detectors: records are detector outcomes (XOR of the listed
    measurements), here checked against the measurement records of the same
    compat-RNG run."""
    circ = "X_ERROR(0.3) 0 1 2\nM 0 1 2\n"
    inp = tmp_path / "c.stim"
    inp.write_text(circ)
    det = tmp_path / "d.txt"
    det.write_text("0 1\n1 2\n0 1 2\n\n2\n")
    common = ["sample", "--in", str(inp), "--shots", "300", "--seed", "5", "--rng", "compat"]
    m = run_cli(common)
    d = run_cli(common + ["--detectors", str(det)])
    assert m.returncode == 0 and d.returncode == 0, d.stderr
    ml = m.stdout.decode().split()
    dl = d.stdout.decode().split()
    assert len(ml) == len(dl) == 300
    for a, b in zip(ml, dl):
        x = [int(c) for c in a]
        assert b == f"{x[0] ^ x[1]}{x[1] ^ x[2]}{x[0] ^ x[1] ^ x[2]}{x[2]}"


def test_bench_csv():
    """cmd_bench (cliffsym.cpp:243-278): CSV header and one row per family
    and size, in the reference's column order."""
    r = run_cli(["bench", "--n", "40", "60", "--family", "all", "--shots", "5000"])
    assert r.returncode == 0, r.stderr
    lines = r.stdout.decode().splitlines()
    assert lines[0] == "family,n,init_seconds,sampling_seconds,shots"
    rows = [line.split(",") for line in lines[1:]]
    assert [(f, n) for f, n, *_ in rows] == [(f, n) for f in ("sparse_cnot", "dense_cnot",
                                                                "dense_cnot_depolarize")
                                             for n in ("40", "60")]
    assert all(float(r_[2]) >= 0 and float(r_[3]) > 0 and r_[4] == "5000" for r_ in rows)
