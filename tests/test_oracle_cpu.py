"""The CPU oracle (oracle/symphase_oracle.c) pinned against the reference:
golden vectors of the reference test suite and fixtures produced by the
reference library itself (tests/golden/make_golden.py)."""
import json

import numpy as np
import pytest

from conftest import golden_circuit


def test_mix64_and_keyed_draw_definition(port):
    # sampler.hpp:14-26 restated in Python integers.
    M = (1 << 64) - 1

    def mix(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)

    for seed, g, s in [(0, 0, 0), (42, 1, 0), (42, 7, 123456), (M, M, M), (9, 3, 1 << 40)]:
        assert port.L.orc_mix64(seed) == mix(seed)
        assert port.L.orc_keyed_draw(seed, g, s) == mix(mix(mix(seed) ^ g) ^ s)
    assert port.L.orc_unit_double(M) == (M >> 11) * 2.0 ** -53


def test_group_bits_semantics(port):
    # fill_group (sampler.cpp:11-44): DEP1 identity below 1-p, then X, Z, Y.
    u_of = lambda v: int(v * 2 ** 53) << 11  # noqa: E731
    p = 0.3
    assert port.L.orc_group_bits(3, p, u_of(0.69)) == 0
    assert port.L.orc_group_bits(3, p, u_of(0.71)) == 1
    assert port.L.orc_group_bits(3, p, u_of(0.81)) == 2
    assert port.L.orc_group_bits(3, p, u_of(0.91)) == 3
    assert port.L.orc_group_bits(4, p, u_of(0.999999)) == 15
    assert port.L.orc_group_bits(1, 1.0, (1 << 64) - 1) == 1
    assert port.L.orc_group_bits(1, 0.0, 0) == 0
    assert port.L.orc_group_bits(2, 0.5, 3) == 1


@pytest.mark.parametrize("case", ["worked.700.42", "mixed.200.9", "degen.500.99", "dep.1000.42",
                                  "rep5.777.1", "surf3.1500.2024", "rand3.64.7", "rand5.513.5"])
def test_port_draw_matches_reference_draw_assignments(port, golden, case):
    name, n, seed = case.split(".")
    _, init = golden_circuit(golden, name)
    S = port.draw_assignments(init, int(n), int(seed))
    assert np.array_equal(S, golden["draws"][case])


@pytest.mark.parametrize("case", ["worked.700.42", "mixed.200.9", "degen.500.99", "dep.1000.42",
                                  "rep5.777.1", "surf3.1500.2024", "rand3.64.7", "rand5.513.5",
                                  "det_m0.3.0"])
@pytest.mark.parametrize("fmt", ["01", "b8"])
def test_port_end_to_end_matches_cmd_sample(port, golden, case, fmt):
    name, n, seed = case.split(".")
    n, seed = int(n), int(seed)
    _, init = golden_circuit(golden, name)
    S = port.draw_assignments(init, n, seed)
    m = port.sample(init.row_ptr, init.sym_idx, S, n)
    got = port.encode(m, init.n_meas, n, fmt)
    assert got == golden["cmd_sample"][f"{case}.{fmt}"].tobytes()


def test_port_sample_matches_reference_on_supplied_batches(port, golden):
    g = golden["given_s"]
    for i in range(int(g["count"][0])):
        n = int(g[f"{i}.n"][0])
        out = port.sample(g[f"{i}.row_ptr"], g[f"{i}.sym_idx"], g[f"{i}.S"], n)
        assert np.array_equal(out, g[f"{i}.out"]), i


def test_encode_golden_vectors(port):
    # test_sampler.cpp:120-147
    m = np.array([[1], [0], [1]], dtype=np.uint64)
    assert port.encode(m, 3, 1, "01") == b"101\n"
    assert port.encode(m, 3, 1, "b8") == bytes([0x05])
    nine = np.ones((9, 1), dtype=np.uint64)
    assert port.encode(nine, 9, 1, "b8") == bytes([0xFF, 0x01])
    empty = np.zeros((0, 0), dtype=np.uint64)
    assert port.encode(empty, 0, 0, "01") == b""
    assert port.encode(empty, 0, 0, "b8") == b""
    # test_cli.cpp:117-122: `M 0`, 3 shots -> "0\n0\n0\n"
    z = np.zeros((1, 1), dtype=np.uint64)
    assert port.encode(z, 1, 3, "01") == b"0\n0\n0\n"


def test_sample_out_of_range_symbol(port):
    # test_sampler.cpp:114-118: expression {5} against a 3-symbol batch throws out_of_range.
    with pytest.raises(IndexError):
        port.sample(np.array([0, 1], np.uint64), np.array([5], np.uint32),
                    np.zeros((3, 1), np.uint64), 8)


def test_draw_zero_shots_rejected(port, golden):
    _, init = golden_circuit(golden, "worked")
    with pytest.raises(ValueError):
        port.draw_assignments(init, 0, 1)


def test_port_vs_live_reference_random(port, ref):
    """Port == reference on fresh random inputs (only where oracle/_ref is built)."""
    from paper_2311_03906_b200 import circuits as CI
    rng = CI.MT19937_64(99)
    for _ in range(10):
        text = CI.random_test_circuit(rng, n_qubits=1 + rng.below(5), n_instr=10 + rng.below(40))
        c = ref.circuit(text)
        n, seed = 1 + rng.below(900), rng()
        from paper_2311_03906_b200.sampler import GROUP_DTYPE, InitResult
        groups = np.zeros(c.n_groups, dtype=GROUP_DTYPE)
        groups["dist"], groups["param"] = c.dist, c.param
        groups["first_symbol"], groups["arity"] = c.first, c.arity
        init = InitResult(c.n_qubits, c.n_sym, c.row_ptr, c.sym_idx, groups)
        S = port.draw_assignments(init, n, seed)
        assert np.array_equal(S, c.draw(n, seed))
        m = port.sample(c.row_ptr, c.sym_idx, S, n)
        assert port.encode(m, c.n_meas, n, "b8") == c.sample_encode(n, seed, "b8")


def test_golden_fixture_index(golden):
    names = json.loads(str(golden["frontend"]["names"]))
    assert "worked" in names and "surf3" in names


def test_cfg5_generator_shapes():
    """cfg5 rows: ascending symbol ids in [1, v], density within 5 sigma."""
    from paper_2311_03906_b200 import circuits as CI
    for dens in CI.CFG5_DENSITIES:
        m, v = 200, 4000
        rp, si = CI.random_msym_rows(m, v, dens, seed=7)
        assert rp[0] == 0 and len(rp) == m + 1
        for k in range(m):
            r = si[rp[k]:rp[k + 1]]
            assert np.all(np.diff(r.astype(np.int64)) > 0) and (len(r) == 0 or (r[0] >= 1 and r[-1] <= v))
        n = m * v
        assert abs(int(rp[-1]) - n * dens) <= 5 * (n * dens * (1 - dens)) ** 0.5 + 1
        rp2, si2 = CI.random_msym_rows(m, v, dens, seed=7)
        assert np.array_equal(rp, rp2) and np.array_equal(si, si2)
