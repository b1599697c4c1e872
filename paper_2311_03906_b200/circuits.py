"""Synthetic circuit generators for the BASELINE.json configurations.

The reference ships none of these workloads (its own generators,
circuit_gen.cpp:56-106, are the paper's Fig. 3 families), so these follow
SURVEY.md Appendix A. All circuits use only instructions the reference parser
accepts (circuit.cpp:51-69): H S S_DAG X Y Z CX M R X_ERROR Y_ERROR Z_ERROR
DEPOLARIZE1 DEPOLARIZE2 TICK.
"""
from __future__ import annotations

from dataclasses import dataclass


class MT19937_64:
    """std::mt19937_64 (the reference's test RNG), for seeded generators."""

    _N, _M = 312, 156
    _MATRIX_A = 0xB5026F5AA96619E9
    _UM, _LM = 0xFFFFFFFF80000000, 0x7FFFFFFF
    _MASK = (1 << 64) - 1

    def __init__(self, seed: int = 5489):
        self.mt = [0] * self._N
        self.mt[0] = seed & self._MASK
        for i in range(1, self._N):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & self._MASK
        self.idx = self._N

    def _twist(self):
        mt, N, M = self.mt, self._N, self._M
        for i in range(N):
            x = (mt[i] & self._UM) | (mt[(i + 1) % N] & self._LM)
            xa = x >> 1
            if x & 1:
                xa ^= self._MATRIX_A
            mt[i] = mt[(i + M) % N] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self._N:
            self._twist()
        x = self.mt[self.idx]
        self.idx += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & self._MASK

    def below(self, n: int) -> int:
        """Uniform integer in [0, n) by rejection (no modulo bias)."""
        lim = (1 << 64) - ((1 << 64) % n)
        while True:
            v = self()
            if v < lim:
                return v % n


def _fmt(name, targets, p=None):
    head = name if p is None else f"{name}({p!r})"
    return head + " " + " ".join(str(t) for t in targets)


def repetition_code(distance: int = 5, rounds: int = 5, p: float = 0.01) -> str:
    """BASELINE config 1: data on even, ancillas on odd qubits."""
    data = [2 * i for i in range(distance)]
    anc = [2 * i + 1 for i in range(distance - 1)]
    left = [(2 * i, 2 * i + 1) for i in range(distance - 1)]
    right = [(2 * i + 2, 2 * i + 1) for i in range(distance - 1)]
    out = []
    for _ in range(rounds):
        out.append(_fmt("R", anc))
        out.append(_fmt("X_ERROR", anc, p))
        for pairs in (left, right):
            flat = [q for pr in pairs for q in pr]
            out.append(_fmt("CX", flat))
            out.append(_fmt("DEPOLARIZE2", flat, p))
        out.append(_fmt("X_ERROR", anc, p))
        out.append(_fmt("M", anc))
    out.append(_fmt("X_ERROR", data, p))
    out.append(_fmt("M", data))
    return "\n".join(out) + "\n"


@dataclass
class SurfaceLayout:
    data: list
    xanc: list
    zanc: list
    index: dict


def surface_layout(d: int) -> SurfaceLayout:
    data = [(x, y) for x in range(1, 2 * d, 2) for y in range(1, 2 * d, 2)]
    dset = set(data)
    xanc, zanc = [], []
    for x in range(0, 2 * d + 1, 2):
        for y in range(0, 2 * d + 1, 2):
            is_x = ((x + y) // 2) % 2 == 0
            nb = sum((x + dx, y + dy) in dset for dx in (-1, 1) for dy in (-1, 1))
            boundary = (y in (0, 2 * d)) if is_x else (x in (0, 2 * d))
            if nb == 4 or (nb == 2 and boundary):
                (xanc if is_x else zanc).append((x, y))
    order = data + xanc + zanc
    return SurfaceLayout(data, xanc, zanc, {c: i for i, c in enumerate(order)})


def surface_code(d: int = 5, rounds: int | None = None, p: float = 1e-3) -> str:
    """BASELINE configs 2/3: rotated surface-code memory-Z."""
    rounds = d if rounds is None else rounds
    L = surface_layout(d)
    ix = L.index
    dset = set(L.data)
    data = [ix[c] for c in L.data]
    xa = [ix[c] for c in L.xanc]
    za = [ix[c] for c in L.zanc]
    anc = xa + za
    allq = sorted(ix.values())
    x_off = [(1, 1), (-1, 1), (1, -1), (-1, -1)]
    z_off = [(1, 1), (1, -1), (-1, 1), (-1, -1)]
    layers = []
    for l in range(4):
        pairs = []
        for (x, y) in L.xanc:
            nb = (x + x_off[l][0], y + x_off[l][1])
            if nb in dset:
                pairs.append((ix[(x, y)], ix[nb]))
        for (x, y) in L.zanc:
            nb = (x + z_off[l][0], y + z_off[l][1])
            if nb in dset:
                pairs.append((ix[nb], ix[(x, y)]))
        layers.append(pairs)
    out = []
    for _ in range(rounds):
        out.append(_fmt("R", anc))
        out.append(_fmt("X_ERROR", anc, p))
        out.append(_fmt("DEPOLARIZE1", data, p))
        out.append(_fmt("H", xa))
        out.append(_fmt("DEPOLARIZE1", allq, p))
        for pairs in layers:
            flat = [q for pr in pairs for q in pr]
            busy = set(flat)
            out.append(_fmt("CX", flat))
            out.append(_fmt("DEPOLARIZE2", flat, p))
            idle = [q for q in allq if q not in busy]
            if idle:
                out.append(_fmt("DEPOLARIZE1", idle, p))
        out.append(_fmt("H", xa))
        out.append(_fmt("DEPOLARIZE1", allq, p))
        out.append(_fmt("X_ERROR", anc, p))
        out.append(_fmt("M", anc))
        out.append(_fmt("DEPOLARIZE1", data, p))
    out.append(_fmt("X_ERROR", data, p))
    out.append(_fmt("M", data))
    return "\n".join(out) + "\n"


def surface_code_detectors(d: int = 5, rounds: int | None = None):
    """Detectors and the logical observable of `surface_code(d, rounds)`
    (memory-Z), as lists of measurement indices (the
    reference has no DETECTOR instruction, so these are builder-defined).

    Record order per round is X ancillas then Z ancillas (`M anc`), then the
    final data measurements. Z stabilizers: round 0 alone (deterministic),
    then round r xor r-1, then the last round xor the data on the support.
    X stabilizers: round r xor r-1 for r >= 1 (round 0 is random). The
    observable is the data row y = 1 (a logical Z: it commutes with every X
    stabilizer, so it is deterministic without noise)."""
    rounds = d if rounds is None else rounds
    L = surface_layout(d)
    dset = set(L.data)
    nx, nz = len(L.xanc), len(L.zanc)
    na = nx + nz
    data_pos = {c: k for k, c in enumerate(L.data)}
    dets = []
    for r in range(rounds):
        for j in range(nx):
            if r >= 1:
                dets.append([r * na + j, (r - 1) * na + j])
        for j in range(nz):
            i = nx + j
            dets.append([i] if r == 0 else [r * na + i, (r - 1) * na + i])
    for j, (x, y) in enumerate(L.zanc):
        sup = [(x + dx, y + dy) for dx in (-1, 1) for dy in (-1, 1) if (x + dx, y + dy) in dset]
        dets.append([(rounds - 1) * na + nx + j] + [rounds * na + data_pos[c] for c in sup])
    obs = [[rounds * na + data_pos[c] for c in L.data if c[1] == 1]]
    return dets, obs


def random_clifford(n: int = 1000, layers: int = 100, p: float = 1e-3, seed: int = 1,
                    measure_every: int = 10, measure_frac: float = 0.1) -> str:
    """BASELINE config 4: layered random Clifford circuit."""
    rng = MT19937_64(seed)
    out = []
    for layer in range(1, layers + 1):
        hs, ss = [], []
        for q in range(n):
            if rng() & 1:
                (hs if rng() & 1 else ss).append(q)
        if hs:
            out.append(_fmt("H", hs))
        if ss:
            out.append(_fmt("S", ss))
        perm = list(range(n))
        for i in range(n - 1, 0, -1):
            j = rng.below(i + 1)
            perm[i], perm[j] = perm[j], perm[i]
        flat = []
        for i in range(0, n - 1, 2):
            a, b = perm[i], perm[i + 1]
            if rng() & 1:
                a, b = b, a
            flat += [a, b]
        if flat:
            out.append(_fmt("CX", flat))
        out.append(_fmt("DEPOLARIZE1", range(n), p))
        if layer % measure_every == 0 and layer < layers:
            k = max(1, int(round(measure_frac * n)))
            pool = list(range(n))
            for i in range(k):
                j = i + rng.below(n - i)
                pool[i], pool[j] = pool[j], pool[i]
            out.append(_fmt("M", sorted(pool[:k])))
    out.append(_fmt("M", range(n)))
    return "\n".join(out) + "\n"


def random_test_circuit(rng: MT19937_64, n_qubits: int = 4, n_instr: int = 40,
                        noise: bool = True, resets: bool = True) -> str:
    """Random mixed circuits exercising every instruction kind (for parity tests)."""
    kinds = ["H", "S", "S_DAG", "X", "Y", "Z", "CX", "M", "TICK"]
    if resets:
        kinds.append("R")
    if noise:
        kinds += ["X_ERROR", "Y_ERROR", "Z_ERROR", "DEPOLARIZE1", "DEPOLARIZE2"]
    probs = [0.0, 0.01, 0.1, 0.25, 0.5, 1.0]
    out = []
    for _ in range(n_instr):
        k = kinds[rng.below(len(kinds))]
        if k == "TICK":
            out.append("TICK")
            continue
        if k in ("CX", "DEPOLARIZE2"):
            if n_qubits < 2:
                continue
            npairs = 1 + rng.below(2)
            flat = []
            for _ in range(npairs):
                a = rng.below(n_qubits)
                b = (a + 1 + rng.below(n_qubits - 1)) % n_qubits
                flat += [a, b]
            tg = flat
        else:
            tg = [rng.below(n_qubits) for _ in range(1 + rng.below(3))]
        p = probs[rng.below(len(probs))] if k.endswith("ERROR") or k.startswith("DEPOL") else None
        out.append(_fmt(k, tg, p))
    out.append(_fmt("M", range(n_qubits)))
    return "\n".join(out) + "\n"


CONFIGS = {
    "cfg1": dict(name="repetition d=5, 5 rounds", text=lambda: repetition_code(5, 5, 0.01),
                 shots=10**6),
    "cfg2": dict(name="rotated surface d=5, 5 rounds, p=1e-3",
                 text=lambda: surface_code(5, 5, 1e-3), shots=10**7),
    "cfg3": dict(name="rotated surface d=15, 15 rounds, p=1e-3",
                 text=lambda: surface_code(15, 15, 1e-3), shots=10**8),
    "cfg4": dict(name="random Clifford n=1000, 100 layers",
                 text=lambda: random_clifford(1000, 100, 1e-3, 1), shots=10**6),
}


# ---- cfg5: raw GF(2) sampling sweep (BASELINE.json configs[4]) -------------
#
# Not a circuit: M_sym itself is drawn, m rows x v fault variables with
# i.i.d. Bernoulli(dens) entries (geometric gaps for dens <
# 0.05, else per-entry bits; seed 7), and each variable is its own
# Bernoulli(p) fault group. Symbol 0 is the constant s0 (unused by the rows),
# symbols 1..v the faults, as the reference registry would number them
# (symbols.hpp:49-71).
CFG5_DENSITIES = (0.001, 0.01, 0.5)
CFG5_RATES = (1e-4, 1e-3, 1e-2)


BENCH_FAMILIES = {"a": "sparse_cnot", "b": "dense_cnot", "c": "dense_cnot_depolarize"}


def bench_family(family: str, n: int, seed: int = 0, noise_p: float = 1e-3) -> str:
    """The paper's Fig. 3 scaling families as `cliffsym bench` builds them
    (circuit_gen.cpp:19-66): n qubits, n layers; each layer applies H or S or
    nothing to every qubit (1/3 each), CX on 5 random pairs (sparse_cnot) or
    on a random perfect matching of all qubits (dense_cnot*), DEPOLARIZE1(p)
    on every qubit (dense_cnot_depolarize), and Z-measures max(1, n/20)
    random qubits; all qubits are measured at the end. Seeded with our own
    MT19937-64 and Fisher-Yates shuffles (same structure and distributions,
    not the reference's exact gate list)."""
    name = BENCH_FAMILIES.get(family, family)
    rng = MT19937_64(seed)
    qubits = list(range(n))

    def shuffle():
        for i in range(n - 1, 0, -1):
            j = rng.below(i + 1)
            qubits[i], qubits[j] = qubits[j], qubits[i]

    pairs = min(5, n // 2) if name == "sparse_cnot" else n // 2
    per_layer = max(1, n // 20)
    lines = []
    for _ in range(n):
        h, s = [], []
        for q in range(n):
            r = rng.below(3)
            (h if r == 0 else s if r == 1 else []).append(q)
        if h:
            lines.append(_fmt("H", h))
        if s:
            lines.append(_fmt("S", s))
        shuffle()
        if pairs:
            lines.append(_fmt("CX", qubits[: 2 * pairs]))
        if name == "dense_cnot_depolarize":
            lines.append(_fmt("DEPOLARIZE1", range(n), noise_p))
        shuffle()
        lines.append(_fmt("M", sorted(qubits[:per_layer])))
    lines.append(_fmt("M", range(n)))
    return "\n".join(lines) + "\n"


def gate_padding_pair(n: int = 32, rounds: int = 6, extra_gates: int = 100_000,
                      seed: int = 0xC8) -> tuple[str, str]:
    """The reference's acceptance criterion C8 workload (acceptance.cpp:437-533):
    a noisy 32-qubit circuit (H on all, CX pairs q / q + n/2, X_ERROR(0.01),
    DEPOLARIZE1(0.02), M all, six rounds), and the same circuit with
    `extra_gates` gates inserted as adjacent self-inverse pairs (H H, CX CX,
    S S_DAG), so every original instruction sees the same state and M_sym is
    unchanged. Returns (base, padded) circuit texts."""
    rng = MT19937_64(seed)
    base = []
    for _ in range(rounds):
        base.append(_fmt("H", range(n)))
        base.append(_fmt("CX", [t for q in range(n // 2) for t in (q, q + n // 2)]))
        base.append(_fmt("X_ERROR", range(n), 0.01))
        base.append(_fmt("DEPOLARIZE1", range(n), 0.02))
        base.append(_fmt("M", range(n)))
    padded, emitted = [], 0

    def pair():
        q = rng.below(n)
        kind = rng.below(3)
        if kind == 0:
            padded.extend([f"H {q}", f"H {q}"])
        elif kind == 1:
            b = rng.below(n)
            while b == q:
                b = rng.below(n)
            padded.extend([f"CX {q} {b}", f"CX {q} {b}"])
        else:
            padded.extend([f"S {q}", f"S_DAG {q}"])

    per_slot = extra_gates // 2 // len(base)
    for inst in base:
        for _ in range(per_slot):
            pair()
            emitted += 1
        padded.append(inst)
    while 2 * emitted < extra_gates:
        pair()
        emitted += 1
    return "\n".join(base) + "\n", "\n".join(padded) + "\n"


def random_msym_rows(m: int, v: int, dens: float, seed: int = 7):
    """CSR rows (row_ptr u64 [m+1], sym_idx u32 ascending in [1, v])."""
    import numpy as np

    rng = np.random.default_rng(seed)
    rows = []
    if dens < 0.05:
        # geometric gaps: positions of successes in a Bernoulli(dens) row
        for _ in range(m):
            need = int(v * dens + 8 * (v * dens) ** 0.5 + 16)
            pos = np.cumsum(rng.geometric(dens, size=need)) - 1
            while pos[-1] < v:  # rare: extend
                more = np.cumsum(rng.geometric(dens, size=need)) + pos[-1]
                pos = np.concatenate([pos, more])
            rows.append((pos[pos < v] + 1).astype(np.uint32))
    else:
        for _ in range(m):
            bits = rng.random(v) < dens
            rows.append((np.flatnonzero(bits) + 1).astype(np.uint32))
    row_ptr = np.zeros(m + 1, dtype=np.uint64)
    row_ptr[1:] = np.cumsum([len(r) for r in rows])
    sym_idx = np.concatenate(rows) if rows else np.zeros(0, np.uint32)
    return row_ptr, sym_idx


def random_msym_model(m: int = 10**4, v: int = 10**5, dens: float = 0.001, p: float = 1e-3,
                      seed: int = 7):
    """cfg5 model as an InitResult: random rows + v Bernoulli(p) groups."""
    import numpy as np

    from .sampler import GROUP_DTYPE, InitResult

    row_ptr, sym_idx = random_msym_rows(m, v, dens, seed)
    return InitResult(0, v + 1, row_ptr, sym_idx, bernoulli_groups(v, p))


def bernoulli_groups(v: int, p: float):
    """Group table: s0 (constant) + v single-symbol Bernoulli(p) groups."""
    import numpy as np

    from .sampler import GROUP_DTYPE

    groups = np.zeros(v + 1, dtype=GROUP_DTYPE)
    groups["dist"][1:] = 1  # Bernoulli
    groups["param"][1:] = p
    groups["first_symbol"] = np.arange(v + 1, dtype=np.uint32)
    groups["arity"] = 1
    return groups
