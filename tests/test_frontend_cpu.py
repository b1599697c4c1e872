"""Host front end (native parse + symbolic pass, CPU-only code in
libsymphase_b200.so) against the reference's run_initialization."""
import json

import numpy as np
import pytest

from conftest import golden_circuit
from paper_2311_03906_b200 import circuits as CI
from paper_2311_03906_b200 import run_initialization
from paper_2311_03906_b200._native import LogicError, ParseError  # noqa: F401


def _same(a, b):
    return (a.n_sym == b.n_sym and np.array_equal(a.row_ptr, b.row_ptr)
            and np.array_equal(a.sym_idx, b.sym_idx)
            and np.array_equal(a.groups["dist"], b.groups["dist"])
            and np.array_equal(a.groups["param"], b.groups["param"])
            and np.array_equal(a.groups["first_symbol"], b.groups["first_symbol"])
            and np.array_equal(a.groups["arity"], b.groups["arity"]))


def test_golden_expressions_and_registry(golden):
    names = json.loads(str(golden["frontend"]["names"]))
    for name in names:
        text, want = golden_circuit(golden, name)
        got = run_initialization(text)
        assert _same(got, want), name


def test_worked_example_expressions():
    # acceptance.cpp:110-138: m1 = s3, m2 = s1 ^ s2 ^ s3 (0-based ids here).
    init = run_initialization("H 0\nCX 0 1\nX_ERROR(0.1) 0 1\nM 0 1\n")
    assert init.expressions == [[3], [1, 2, 3]]


def test_four_qubit_example():
    # acceptance.cpp:141-177: m = s1, s2, s2^s3, s3^s4
    text = ("H 0\nCX 0 1\nCX 1 2\nCX 2 3\nZ_ERROR(0.1) 0\nX_ERROR(0.1) 1\nX_ERROR(0.1) 2\n"
            "X_ERROR(0.1) 3\nCX 2 3\nCX 1 2\nCX 0 1\nH 0\nM 0 1 2 3\n")
    assert run_initialization(text).expressions == [[1], [2], [2, 3], [3, 4]]


def test_noise_symbol_numbering():
    # test_sampler.cpp:193-196: three X_ERRORs on qubit 0 -> m = s1 ^ s2 ^ s3
    init = run_initialization("X_ERROR(0.05) 0\nX_ERROR(0.2) 0\nX_ERROR(0.45) 0\nM 0\n")
    assert init.expressions == [[1, 2, 3]]
    assert init.n_sym == 4


def test_constant_symbol_rows():
    # test_sampler.cpp:36-46: X 0; M 0; M 0 -> both rows {s0}, registry size 1
    init = run_initialization("X 0\nM 0\nM 0\n")
    assert init.expressions == [[0], [0]]
    assert init.n_sym == 1


def test_empty_circuit():
    init = run_initialization("")
    assert init.n_meas == 0 and init.n_sym == 1 and len(init.groups) == 1


@pytest.mark.parametrize("text,line", [("H 0\nFROB 1\n", 2), ("M 0\nX_ERROR 0\n", 2),
                                       ("H(0.1) 0\n", 1), ("CX 0 0\n", 1), ("CX 0\n", 1),
                                       ("TICK 3\n", 1), ("M\n", 1), ("X_ERROR(1.5) 0\n", 1),
                                       ("X_ERROR(0.1 0\n", 1), ("M -1\n", 1),
                                       ("\n\nREPEAT 3 {\n", 3), ("DETECTOR rec[-1]\n", 1)])
def test_parse_errors_carry_line_numbers(text, line):
    with pytest.raises(ParseError) as e:
        run_initialization(text)
    assert f"line {line}:" in str(e.value)


def test_parse_accepts_aliases_case_comments():
    # test_circuit.cpp:38-53
    init = run_initialization("# c\n  h 5   # t\n\ncnot 0 1\nmz 2\ntick\n")
    assert init.n_qubits == 6 and init.n_meas == 1


def test_generator_shapes_match_survey():
    # SURVEY.md §8 table, measured from the reference's own pass.
    rep = run_initialization(CI.repetition_code(5, 5, 0.01))
    assert (rep.n_meas, rep.n_sym, rep.nnz) == (25, 206, 280)
    s5 = run_initialization(CI.surface_code(5, 5, 1e-3))
    assert (s5.n_meas, s5.n_sym, s5.nnz) == (145, 3730, 12569)


def test_frontend_matches_live_reference_random(ref):
    rng = CI.MT19937_64(4242)
    for _ in range(150):
        text = CI.random_test_circuit(rng, n_qubits=1 + rng.below(7), n_instr=5 + rng.below(70))
        c = ref.circuit(text)
        got = run_initialization(text)
        assert got.n_sym == c.n_sym
        assert np.array_equal(got.row_ptr, c.row_ptr)
        assert np.array_equal(got.sym_idx, c.sym_idx)
        assert np.array_equal(got.groups["dist"], c.dist)
        assert np.array_equal(got.groups["first_symbol"], c.first)


def test_frontend_matches_live_reference_surface9(ref):
    text = CI.surface_code(9, 9, 1e-3)
    c = ref.circuit(text)
    got = run_initialization(text)
    assert np.array_equal(got.row_ptr, c.row_ptr) and np.array_equal(got.sym_idx, c.sym_idx)


def test_gate_padding_keeps_expressions(ref):
    """Acceptance C8 (acceptance.cpp:437-533), first half: 100,000 extra gates
    in self-inverse pairs leave M_sym and the registry unchanged — through
    our front end, and equal to the reference library's own pass."""
    base, padded = CI.gate_padding_pair()
    ib, ip = run_initialization(base), run_initialization(padded)
    assert _same(ib, ip)
    c = ref.circuit(padded)
    assert np.array_equal(ip.row_ptr, c.row_ptr) and np.array_equal(ip.sym_idx, c.sym_idx)


def test_bench_families_shape(ref):
    """The Fig. 3 families (circuit_gen.cpp:19-66): n layers of single-qubit
    gates, CX pairs, optional DEPOLARIZE1, max(1, n/20) measurements per layer
    and n at the end; our front end agrees with the reference library."""
    for fam, n in (("a", 40), ("b", 60), ("c", 30), ("b", 130)):
        text = CI.bench_family(fam, n, seed=3)
        init = run_initialization(text)
        assert init.n_meas == n * max(1, n // 20) + n
        c = ref.circuit(text)
        assert np.array_equal(init.row_ptr, c.row_ptr) and np.array_equal(init.sym_idx, c.sym_idx)
    assert "DEPOLARIZE1" in CI.bench_family("c", 20) and "DEPOLARIZE1" not in CI.bench_family("b", 20)


def test_frontend_matches_live_reference_wide_random(ref):
    """Random circuits over 60-200 qubits (several 64-bit words per tableau
    row and column, resets, noise, mid-circuit measurements): the qubit-major
    gate path and its transposes agree with the reference's pass."""
    rng = CI.MT19937_64(9090)
    for _ in range(12):
        n = 60 + rng.below(141)
        text = CI.random_test_circuit(rng, n_qubits=n, n_instr=200 + rng.below(400))
        c = ref.circuit(text)
        got = run_initialization(text)
        assert got.n_sym == c.n_sym
        assert np.array_equal(got.row_ptr, c.row_ptr) and np.array_equal(got.sym_idx, c.sym_idx)


def test_row_form_gate_layers_match_reference(ref):
    """Gate instructions right after measurements run in the row-major form
    (masked sweep for H/S/S_DAG, per pair for CX) while cheaper than a layout
    conversion; repeated qubits and long CX layers go the qubit-major way.
    Layers mixing all of these, with noise and resets, agree with the
    reference's pass."""
    rng = CI.MT19937_64(6060)
    for n in (70, 130, 200):
        qs = list(range(n))
        lines = []

        def subset(frac):
            return [q for q in qs if rng.below(1000) < frac * 1000]

        for layer in range(12):
            for name in ("H", "S_DAG", "S"):
                t = subset(0.4)
                if t and layer % 3 == 2:
                    t = t + t[:1]  # a repeated qubit
                if t:
                    lines.append(f"{name} " + " ".join(map(str, t)))
            for i in range(n - 1, 0, -1):
                j = rng.below(i + 1)
                qs[i], qs[j] = qs[j], qs[i]
            k = 3 if layer % 2 else n // 2
            lines.append("CX " + " ".join(map(str, qs[: 2 * k])))
            qs.sort()
            lines.append("DEPOLARIZE1(0.01) " + " ".join(map(str, subset(0.3) or [0])))
            lines.append("M " + " ".join(map(str, subset(0.2) or [1])))
            if layer % 4 == 1:
                lines.append("R " + " ".join(map(str, subset(0.1) or [2])))
        lines.append("M " + " ".join(map(str, range(n))))
        text = "\n".join(lines) + "\n"
        c = ref.circuit(text)
        got = run_initialization(text)
        assert got.n_sym == c.n_sym
        assert np.array_equal(got.row_ptr, c.row_ptr) and np.array_equal(got.sym_idx, c.sym_idx)


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg4"])
def test_baseline_workloads_match_reference_pass(cfg):
    """cfg2-cfg4 are too large to store: tests/golden/large.json holds sha256
    digests of the reference pass's arrays (make_golden.py large); the
    circuit text is pinned by its digest too."""
    import hashlib
    from pathlib import Path
    want = json.loads((Path(__file__).resolve().parent / "golden" / "large.json").read_text())[cfg]
    text = CI.CONFIGS[cfg]["text"]()
    assert hashlib.sha256(text.encode()).hexdigest() == want["text"]["sha256"]
    from test_gpu_large import digest_ok
    assert digest_ok(run_initialization(text), want)


def _fuzz_line(rng):
    names = ["H", "h", "S", "S_DAG", "X", "Y", "Z", "CX", "cnot", "M", "MZ", "R", "TICK", "tick",
             "X_ERROR", "Y_ERROR", "Z_ERROR", "DEPOLARIZE1", "DEPOLARIZE2", "FROB", "REPEAT",
             "DETECTOR", "QUBIT_COORDS"]
    name = names[rng.integers(len(names))]
    r = rng.random()
    if r < 0.5:
        name += f"({rng.choice(['0.1', '0', '1', '1.5', '-0.1', 'x', '', '1e-3', 'nan'])})"
    elif r < 0.55:
        name += "(0.2"
    n = int(rng.integers(0, 5))
    targets = [str(int(rng.integers(0, 4))) if rng.random() < 0.9 else
               rng.choice(["-1", "a", "2x", "rec[-1]"]) for _ in range(n)]
    ws = [" ", "\t", "  ", " \r"]
    line = name + "".join(ws[rng.integers(len(ws))] + t for t in targets)
    if rng.random() < 0.2:
        line += " # note " + rng.choice(["", "H 0", "#"])
    if rng.random() < 0.1:
        line = "   " + line
    return line


def test_parser_agrees_with_reference_parser(ref):
    """The rewritten scanner/validator accepts exactly what the reference's
    parse_circuit (circuit.cpp:79-168) accepts, and reports the same line.
    Single-line programs first (every rule), then multi-line ones."""
    import re
    rng = np.random.default_rng(77)
    texts = [_fuzz_line(rng) for _ in range(600)]
    texts += ["\n".join(_fuzz_line(rng) for _ in range(int(rng.integers(2, 6))))
              for _ in range(200)]
    for text in texts:
        try:
            ref.circuit(text)
            ref_err = None
        except (ValueError, RuntimeError) as e:
            ref_err = str(e)
        try:
            run_initialization(text)
            ours = None
        except ParseError as e:
            ours = str(e)
        except LogicError:
            ours = "logic"
        if ref_err is None:
            assert ours is None, (text, ours)
            continue
        if "line" not in ref_err:  # a logic error of the symbolic pass, not the parser
            assert ours is not None, (text, ref_err)
            continue
        assert ours is not None and ours != "logic", (text, ref_err)
        want = re.search(r"line (\d+)", ref_err).group(1)
        assert f"line {want}:" in ours, (text, ref_err, ours)
