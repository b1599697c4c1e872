"""Generates tests/golden/*.npz from the REFERENCE library (oracle/_ref, built
from /root/reference/proj/core by oracle/Makefile). Run in the build container:

    make -C oracle && python tests/golden/make_golden.py

Fixtures (all produced by the reference's own public API):
  frontend.npz   circuit text -> run_initialization expressions + registry
  draws.npz      draw_assignments(registry, N, seed), bit-sliced
  cmd_sample.npz draw_assignments + sample + encode_shots ('01' and 'b8'),
                 i.e. cliffsym sample --seed S --shots N (cliffsym.cpp:108-113)
  given_s.npz    sample(expressions, batch) on seeded random batches shaped like
                 acceptance.cpp:312-361 (criterion 6) and tile-straddling sizes
  large.json     run_initialization of the BASELINE workloads cfg2-cfg4 (too
                 large to store): sha256 + length of every InitResult array
                 and of the circuit text (`python make_golden.py large`)
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
from paper_2311_03906_b200 import circuits as CI  # noqa: E402

OUT = Path(__file__).resolve().parent
ref = oracle.Ref()

WORKED = "H 0\nCX 0 1\nX_ERROR(0.1) 0 1\nM 0 1\n"             # acceptance.cpp:40
FOUR = ("H 0\nCX 0 1\nCX 1 2\nCX 2 3\n"                          # acceptance.cpp:41-44
        "Z_ERROR(0.1) 0\nX_ERROR(0.1) 1\nX_ERROR(0.1) 2\nX_ERROR(0.1) 3\n"
        "CX 2 3\nCX 1 2\nCX 0 1\nH 0\nM 0 1 2 3\n")
MIXED = ("H 0\nCX 0 1\nDEPOLARIZE1(0.2) 0\nX_ERROR(0.3) 1\n"     # test_cli.cpp:126-128
         "M 0\nR 1\nH 1\nM 1 0\n")
DEGEN = "X_ERROR(1) 0\nX_ERROR(0) 1\nM 0 1\n"                    # test_sampler.cpp:49
DEP = "DEPOLARIZE1(0.2) 0\nH 0\nM 0\nX_ERROR(0.4) 0\nM 0\n"       # test_sampler.cpp:63


def circuits():
    named = {"worked": WORKED, "four": FOUR, "mixed": MIXED, "degen": DEGEN, "dep": DEP,
             "det_m0": "M 0\n", "noiseless": "X 0\nM 0\nM 0\n",
             "rep5": CI.repetition_code(5, 5, 0.01), "surf3": CI.surface_code(3, 3, 0.01)}
    rng = CI.MT19937_64(20241)
    for i in range(24):
        named[f"rand{i}"] = CI.random_test_circuit(rng, n_qubits=1 + rng.below(6),
                                                   n_instr=5 + rng.below(50))
    return named


def frontend(named):
    d = {"names": json.dumps(list(named))}
    for k, text in named.items():
        c = ref.circuit(text)
        d[f"{k}.text"] = np.frombuffer(text.encode(), dtype=np.uint8)
        d[f"{k}.row_ptr"] = c.row_ptr
        d[f"{k}.sym_idx"] = c.sym_idx
        d[f"{k}.dist"] = c.dist
        d[f"{k}.param"] = c.param
        d[f"{k}.first"] = c.first
        d[f"{k}.arity"] = c.arity
        d[f"{k}.n_sym"] = np.array([c.n_sym], dtype=np.uint64)
    np.savez_compressed(OUT / "frontend.npz", **d)


CASES = [("worked", 700, 42), ("mixed", 200, 9), ("degen", 500, 99), ("dep", 1000, 42),
         ("rep5", 777, 1), ("surf3", 1500, 2024), ("rand3", 64, 7), ("rand5", 513, 5)]


def draws(named):
    d = {}
    for name, n, seed in CASES:
        c = ref.circuit(named[name])
        d[f"{name}.{n}.{seed}"] = c.draw(n, seed)
    np.savez_compressed(OUT / "draws.npz", **d)


def cmd_sample(named):
    d = {}
    for name, n, seed in CASES + [("det_m0", 3, 0)]:
        c = ref.circuit(named[name])
        for fmt in ("01", "b8"):
            d[f"{name}.{n}.{seed}.{fmt}"] = np.frombuffer(c.sample_encode(n, seed, fmt),
                                                          dtype=np.uint8)
    np.savez_compressed(OUT / "cmd_sample.npz", **d)


def given_s():
    rng = np.random.default_rng(0xC6)
    d = {}
    shapes = [(50 + int(rng.integers(251)), 100 + int(rng.integers(401)),
               256 + int(rng.integers(1793))) for _ in range(12)]
    shapes += [(17, 40, n) for n in (1, 63, 64, 65, 511, 512, 513, 1024, 1537)]
    for i, (n_m, n_s, n) in enumerate(shapes):
        S = np.zeros((n_s, (n + 63) // 64), dtype=np.uint64)
        bits = rng.integers(0, 2, size=(n_s, n), dtype=np.uint8)
        pad = np.zeros((n_s, S.shape[1] * 64), dtype=np.uint8)
        pad[:, :n] = bits
        S[:] = np.packbits(pad, axis=1, bitorder="little").view(np.uint64)
        rows = []
        for k in range(n_m):
            nnz = int(rng.integers(31)) if k % 7 else int(k % 3 == 0)  # include empty rows
            rows.append(np.unique(rng.integers(0, n_s, size=nnz)).astype(np.uint32))
        row_ptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.uint64)
        sym_idx = np.concatenate(rows).astype(np.uint32) if rows else np.zeros(0, np.uint32)
        out = ref.sample_given(row_ptr, sym_idx, S, n)
        d[f"{i}.S"] = S
        d[f"{i}.row_ptr"] = row_ptr
        d[f"{i}.sym_idx"] = sym_idx
        d[f"{i}.n"] = np.array([n], dtype=np.uint64)
        d[f"{i}.out"] = out
    d["count"] = np.array([len(shapes)])
    np.savez_compressed(OUT / "given_s.npz", **d)


def digest(a) -> dict:
    a = np.ascontiguousarray(a)
    return {"len": int(a.size), "dtype": str(a.dtype),
            "sha256": hashlib.sha256(a.tobytes()).hexdigest()}


def large():
    d = {}
    for cfg in ("cfg2", "cfg3", "cfg4"):
        text = CI.CONFIGS[cfg]["text"]()
        c = ref.circuit(text)  # the reference's own pass (~1 min at cfg3/cfg4)
        d[cfg] = {"text": digest(np.frombuffer(text.encode(), dtype=np.uint8)),
                  "n_meas": int(c.n_meas), "n_sym": int(c.n_sym),
                  "row_ptr": digest(c.row_ptr.astype(np.uint64)),
                  "sym_idx": digest(c.sym_idx.astype(np.uint32)),
                  "dist": digest(c.dist.astype(np.uint8)),
                  "param": digest(c.param.astype(np.float64)),
                  "first": digest(c.first.astype(np.uint32)),
                  "arity": digest(c.arity.astype(np.uint32))}
        print(cfg, d[cfg]["n_meas"], d[cfg]["n_sym"], flush=True)
    (OUT / "large.json").write_text(json.dumps(d, indent=1) + "\n")


if __name__ == "__main__" and sys.argv[1:] == ["large"]:
    large()
elif __name__ == "__main__":
    named = circuits()
    frontend(named)
    draws(named)
    cmd_sample(named)
    given_s()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
