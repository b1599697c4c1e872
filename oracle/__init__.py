"""TEST INFRASTRUCTURE ONLY — CPU oracles for the sampling hot path.

Two oracles, both built by `make -C oracle` (also run by __graft_entry__.build()):

* `Ref` — the unmodified reference library (cliffsym core compiled from
  /root/reference/proj/core/src, oracle/Makefile) behind oracle/ref_driver.cpp.
  Built only where /root/reference exists; the .so then travels to the GPU
  box with the repo snapshot.
* `Port` — the plain-C restatement in oracle/symphase_oracle.c (keyed_draw,
  fill_group, draw_assignments, sparse GF(2) product, encode_shots), pinned
  against `Ref` and the reference tests' golden vectors.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package. The product library never
links or calls it.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libcliffsym_ref.so"
PORT_SO = HERE / "_build" / "libsymphase_oracle.so"

_u64, _u32, _i, _p, _d = C.c_uint64, C.c_uint32, C.c_int, C.c_void_p, C.c_double


def _ptr(a):
    return None if a is None else a.ctypes.data


class Port:
    """ctypes wrapper of oracle/symphase_oracle.c."""

    def __init__(self, path: Path = PORT_SO):
        if not path.exists():
            raise RuntimeError(f"{path} not built; run `make -C oracle`")
        L = C.CDLL(str(path))
        L.orc_mix64.restype = _u64
        L.orc_mix64.argtypes = [_u64]
        L.orc_keyed_draw.restype = _u64
        L.orc_keyed_draw.argtypes = [_u64, _u64, _u64]
        L.orc_unit_double.restype = _d
        L.orc_unit_double.argtypes = [_u64]
        L.orc_group_bits.restype = C.c_uint
        L.orc_group_bits.argtypes = [_i, _d, _u64]
        L.orc_draw_assignments.restype = _i
        L.orc_draw_assignments.argtypes = [_u64, _p, _p, _p, _p, _u64, _u64, _u64, _p, _u64]
        L.orc_draw_assignments_range.restype = _i
        L.orc_draw_assignments_range.argtypes = [_u64, _p, _p, _p, _p, _u64, _u64, _u64, _u64,
                                                 _p, _u64]
        L.orc_sample_sparse.restype = _i
        L.orc_sample_sparse.argtypes = [_u64, _p, _p, _u64, _u64, _p, _u64, _p, _u64]
        L.orc_encode.restype = _u64
        L.orc_encode.argtypes = [_u64, _u64, _p, _u64, _i, _p]
        self.L = L

    def draw_assignments(self, init, n_shots: int, seed: int, shot_begin: int = 0) -> np.ndarray:
        g = init.groups
        ld = max((n_shots + 63) // 64, 1)
        S = np.zeros((init.n_sym, ld), dtype=np.uint64)
        dist = np.ascontiguousarray(g["dist"])
        param = np.ascontiguousarray(g["param"])
        first = np.ascontiguousarray(g["first_symbol"])
        arity = np.ascontiguousarray(g["arity"])
        r = self.L.orc_draw_assignments_range(len(g), _ptr(dist), _ptr(param), _ptr(first),
                                              _ptr(arity), init.n_sym, shot_begin, n_shots, seed,
                                              _ptr(S), ld)
        if r == -2:
            raise ValueError("need at least one shot")
        return S

    def sample(self, row_ptr, sym_idx, S: np.ndarray, n_shots: int) -> np.ndarray:
        rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        si = np.ascontiguousarray(sym_idx, dtype=np.uint32)
        if si.size == 0:
            si = np.zeros(1, dtype=np.uint32)
        n_meas = len(rp) - 1
        ld = max((n_shots + 63) // 64, 1)
        out = np.zeros((max(n_meas, 1), ld), dtype=np.uint64)
        S = np.ascontiguousarray(S, dtype=np.uint64)
        r = self.L.orc_sample_sparse(n_meas, _ptr(rp), _ptr(si), S.shape[0], n_shots, _ptr(S),
                                     S.shape[1], _ptr(out), ld)
        if r == -1:
            raise IndexError("symbol id out of range")
        return out[:n_meas]

    def encode(self, m: np.ndarray, n_meas: int, n_shots: int, fmt: str) -> bytes:
        f = 0 if fmt == "01" else 1
        size = n_shots * (n_meas + 1) if f == 0 else n_shots * ((n_meas + 7) // 8)
        buf = np.zeros(max(size, 1), dtype=np.uint8)
        m = np.ascontiguousarray(m, dtype=np.uint64)
        ld = m.shape[1] if m.ndim == 2 and m.size else 1
        if m.size == 0:
            m = np.zeros((1, 1), dtype=np.uint64)
        n = self.L.orc_encode(n_meas, n_shots, _ptr(m), ld, f, _ptr(buf))
        return bytes(buf[:n])


class Ref:
    """ctypes wrapper of the reference library (oracle/ref_driver.cpp)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise RuntimeError(f"{path} not built (needs /root/reference at build time)")
        L = C.CDLL(str(path))
        L.ref_init.restype = _i
        L.ref_init.argtypes = [C.c_char_p, C.POINTER(_p), C.c_char_p, C.c_size_t]
        L.ref_free.argtypes = [_p]
        L.ref_dims.argtypes = [_p] + [C.POINTER(_u64)] * 5
        L.ref_export_rows.argtypes = [_p, _p, _p]
        L.ref_export_groups.argtypes = [_p, _p, _p, _p, _p]
        L.ref_sample_given.restype = _i
        L.ref_sample_given.argtypes = [_u64, _p, _p, _u64, _u64, _p, _u64, _p, _u64, C.c_uint]
        L.ref_gf2_multiply_sparse.restype = _i
        L.ref_gf2_multiply_sparse.argtypes = [_u64, _p, _p, _u64, _u64, _p, _u64, _p, _u64]
        L.ref_draw.restype = _i
        L.ref_draw.argtypes = [_p, _u64, _u64, _p, _u64]
        L.ref_sample_encode.restype = C.c_int64
        L.ref_sample_encode.argtypes = [_p, _u64, _u64, _i, C.c_uint, _p, _u64]
        L.ref_encode.restype = C.c_int64
        L.ref_encode.argtypes = [_u64, _u64, _p, _u64, _i, _p, _u64]
        L.ref_init_model.restype = _i
        L.ref_init_model.argtypes = [_u64, _p, _p, _u64, _p, _p, _p, C.POINTER(_p)]
        L.ref_time.restype = _d
        L.ref_time.argtypes = [_p, _u64, _u64, C.c_uint, _u64, _i]
        self.L = L

    class Circuit:
        def __init__(self, ref: "Ref", text: str | None, model=None):
            self.ref = ref
            h = _p()
            if model is not None:  # explicit expressions + group table (cfg5)
                rp = np.ascontiguousarray(model.row_ptr, dtype=np.uint64)
                si = np.ascontiguousarray(model.sym_idx, dtype=np.uint32)
                if si.size == 0:
                    si = np.zeros(1, dtype=np.uint32)
                g = model.groups
                dist = np.ascontiguousarray(g["dist"], dtype=np.uint8)
                param = np.ascontiguousarray(g["param"], dtype=np.float64)
                arity = np.ascontiguousarray(g["arity"], dtype=np.uint32)
                rc = ref.L.ref_init_model(len(rp) - 1, _ptr(rp), _ptr(si), len(dist), _ptr(dist),
                                          _ptr(param), _ptr(arity), C.byref(h))
                if rc != 0:
                    raise ValueError("ref_init_model failed")
            else:
                err = C.create_string_buffer(512)
                rc = ref.L.ref_init(text.encode(), C.byref(h), err, 512)
                if rc != 0:
                    kind = {1: ValueError, 2: RuntimeError}[rc]
                    raise kind(err.value.decode())
            self.h = h
            d = [_u64() for _ in range(5)]
            ref.L.ref_dims(h, *[C.byref(x) for x in d])
            self.n_meas, self.n_sym, self.n_groups, self.nnz, self.n_qubits = (x.value for x in d)
            self.row_ptr = np.zeros(self.n_meas + 1, dtype=np.uint64)
            si = np.zeros(max(self.nnz, 1), dtype=np.uint32)
            ref.L.ref_export_rows(h, _ptr(self.row_ptr), _ptr(si))
            self.sym_idx = si[:self.nnz]
            self.dist = np.zeros(self.n_groups, dtype=np.uint8)
            self.param = np.zeros(self.n_groups, dtype=np.float64)
            self.first = np.zeros(self.n_groups, dtype=np.uint32)
            self.arity = np.zeros(self.n_groups, dtype=np.uint32)
            ref.L.ref_export_groups(h, _ptr(self.dist), _ptr(self.param), _ptr(self.first),
                                    _ptr(self.arity))

        def __del__(self):
            try:
                self.ref.L.ref_free(self.h)
            except Exception:
                pass

        def draw(self, n_shots: int, seed: int) -> np.ndarray:
            ld = max((n_shots + 63) // 64, 1)
            S = np.zeros((self.n_sym, ld), dtype=np.uint64)
            rc = self.ref.L.ref_draw(self.h, n_shots, seed, _ptr(S), ld)
            if rc == -2:
                raise ValueError("need at least one shot")
            return S

        def sample_encode(self, n_shots: int, seed: int, fmt: str, threads: int = 1) -> bytes:
            f = 0 if fmt == "01" else 1
            size = n_shots * (self.n_meas + 1) if f == 0 else n_shots * ((self.n_meas + 7) // 8)
            buf = np.zeros(max(size, 1), dtype=np.uint8)
            n = self.ref.L.ref_sample_encode(self.h, n_shots, seed, f, threads, _ptr(buf), buf.size)
            if n < 0:
                raise RuntimeError(f"ref_sample_encode failed ({n})")
            return bytes(buf[:n])

        def time(self, total_shots: int, chunk: int, threads: int, seed: int, mode: int) -> float:
            return self.ref.L.ref_time(self.h, total_shots, chunk, threads, seed, mode)

    def circuit(self, text: str) -> "Ref.Circuit":
        return Ref.Circuit(self, text)

    def model(self, init) -> "Ref.Circuit":
        """A reference InitResult from an InitResult-like model (no circuit)."""
        return Ref.Circuit(self, None, model=init)

    def sample_given(self, row_ptr, sym_idx, S: np.ndarray, n_shots: int, threads: int = 1):
        rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        si = np.ascontiguousarray(sym_idx, dtype=np.uint32)
        if si.size == 0:
            si = np.zeros(1, dtype=np.uint32)
        n_meas = len(rp) - 1
        ld = max((n_shots + 63) // 64, 1)
        out = np.zeros((max(n_meas, 1), ld), dtype=np.uint64)
        S = np.ascontiguousarray(S, dtype=np.uint64)
        rc = self.L.ref_sample_given(n_meas, _ptr(rp), _ptr(si), S.shape[0], n_shots, _ptr(S),
                                     S.shape[1], _ptr(out), ld, threads)
        if rc == -1:
            raise IndexError("symbol id out of range")
        if rc != 0:
            raise RuntimeError(f"ref_sample_given failed ({rc})")
        return out[:n_meas]

    def encode(self, m: np.ndarray, n_meas: int, n_shots: int, fmt: str) -> bytes:
        f = 0 if fmt == "01" else 1
        size = n_shots * (n_meas + 1) if f == 0 else n_shots * ((n_meas + 7) // 8)
        buf = np.zeros(max(size, 1), dtype=np.uint8)
        m = np.ascontiguousarray(m, dtype=np.uint64)
        if m.size == 0:
            m = np.zeros((1, 1), dtype=np.uint64)
        n = self.L.ref_encode(n_meas, n_shots, _ptr(m), m.shape[1], f, _ptr(buf), buf.size)
        return bytes(buf[:n])


def have_ref() -> bool:
    return REF_SO.exists()


def flip_rates(init) -> np.ndarray:
    """Analytic P(m_k = 1) for every measurement row (piling-up lemma over
    independent groups; generalises test_sampler.cpp:189-203 to correlated
    DEPOLARIZE groups): P = 1/2 (1 - prod_g (1 - 2 P_g(odd parity))) XOR const."""
    g = init.groups
    sym_group = np.zeros(init.n_sym, dtype=np.int64)
    for gi, (first, ar) in enumerate(zip(g["first_symbol"], g["arity"])):
        sym_group[first:first + ar] = gi
    out = np.zeros(init.n_meas)
    for k in range(init.n_meas):
        syms = init.sym_idx[init.row_ptr[k]:init.row_ptr[k + 1]]
        masks: dict[int, int] = {}
        const = 0
        for s in syms:
            gi = int(sym_group[s])
            if gi == 0:
                const ^= 1
                continue
            masks[gi] = masks.get(gi, 0) | (1 << int(s - g["first_symbol"][gi]))
        prod = 1.0
        for gi, mask in masks.items():
            prod *= 1.0 - 2.0 * _odd_parity_prob(int(g["dist"][gi]), float(g["param"][gi]), mask)
        p1 = 0.5 * (1.0 - prod)
        out[k] = 1.0 - p1 if const else p1
    return out


def _odd_parity_prob(dist: int, p: float, mask: int) -> float:
    """P(XOR of the masked symbols of one group = 1) under fill_group's pmf
    (sampler.cpp:11-44)."""
    if dist in (1,):
        return p
    if dist == 2:
        return 0.5
    if dist == 3:  # patterns 1,2,3 each p/3
        return sum(p / 3 for pat in (1, 2, 3) if bin(pat & mask).count("1") % 2)
    if dist == 4:  # patterns 1..15 each p/15
        return sum(p / 15 for pat in range(1, 16) if bin(pat & mask).count("1") % 2)
    return 0.0
