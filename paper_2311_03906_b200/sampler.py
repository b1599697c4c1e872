"""Host-side mirror of the reference's sampler interface over the C ABI.

Reference interface (cliffsym, proj/core/include/cliffsym):
  parse_circuit(text)                      circuit.hpp:55
  run_initialization(instructions)         tableau.hpp:101  -> InitResult
  draw_assignments(registry, n_smp, seed)  sampler.hpp:51-52
  sample(expressions, batch, threads)      sampler.hpp:57-58
  encode_shots(m, format)                  sampler.hpp:65
  shot_bits(m, shot)                       sampler.hpp:68

Here the symbolic pass runs in the native host library and everything after
it runs on the GPU: `Sampler.sample` is the fused draw+product kernel,
`Sampler.draw_assignments` / `Sampler.sample_given` split it like the
reference does, and `Sampler.encode` is encode_shots. Device buffers are torch
tensors (torch is plumbing: memory, streams, distributed); every bit of
compute goes through libsymphase_b200.so. Results use the bit-sliced layout
of include/symphase_b200.h: int64 words [rows, ceil(n_shots/64)], bit j%64 of
word j/64 of row r = element (r, j).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N

GROUP_DTYPE = np.dtype([("dist", np.uint8), ("reserved", np.uint8, 7), ("param", np.float64),
                        ("first_symbol", np.uint32), ("arity", np.uint32)])
assert GROUP_DTYPE.itemsize == C.sizeof(N.sp_group)

DIST_NAMES = {0: "constant", 1: "bernoulli", 2: "coin", 3: "depolarize1", 4: "depolarize2"}
FORMATS = {"01": 0, "b8": 1}
RNGS = {"philox": 0, "compat": 1}
PRODUCTS = {"auto": 0, "sparse": 1, "dense": 2, "tensor": 3}


def _ptr(a) -> int:
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


@dataclass
class InitResult:
    """InitResult (tableau.hpp:94-99): M_sym rows + the symbol-group registry."""

    n_qubits: int
    n_sym: int
    row_ptr: np.ndarray  # uint64 [n_meas+1]
    sym_idx: np.ndarray  # uint32 [nnz]
    groups: np.ndarray   # GROUP_DTYPE [n_groups]

    @property
    def n_meas(self) -> int:
        return len(self.row_ptr) - 1

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def expressions(self) -> list[list[int]]:
        rp = self.row_ptr
        return [self.sym_idx[rp[k]:rp[k + 1]].tolist() for k in range(self.n_meas)]

    def save(self, path) -> None:
        """On-disk M_sym cache: CSR rows + group table, so a
        large circuit's one-pass init (seconds at d=15) runs once."""
        np.savez_compressed(path, n_qubits=np.array([self.n_qubits]),
                            n_sym=np.array([self.n_sym]), row_ptr=self.row_ptr,
                            sym_idx=self.sym_idx, groups=self.groups.view(np.uint8))

    @classmethod
    def load(cls, path) -> "InitResult":
        z = np.load(path)
        groups = np.ascontiguousarray(z["groups"]).view(GROUP_DTYPE).reshape(-1)
        return cls(int(z["n_qubits"][0]), int(z["n_sym"][0]), z["row_ptr"].astype(np.uint64),
                   z["sym_idx"].astype(np.uint32), groups)

    def detector_model(self, detectors) -> "InitResult":
        """Detector layer: rows = GF(2) sums of the listed measurements' rows
        (D_sym = A . M_sym, sp_detector_rows), same symbols and groups. The
        result samples like any model: detector records and counts."""
        L = N.lib()
        det_ptr = np.zeros(len(detectors) + 1, dtype=np.uint64)
        det_ptr[1:] = np.cumsum([len(d) for d in detectors])
        det_meas = np.ascontiguousarray(np.concatenate(
            [np.asarray(d, dtype=np.uint32) for d in detectors]) if len(detectors) else
            np.zeros(1, np.uint32), dtype=np.uint32)
        if det_meas.size == 0:
            det_meas = np.zeros(1, np.uint32)
        rp = np.zeros(len(detectors) + 1, dtype=np.uint64)
        nnz = C.c_uint64()
        si = np.ascontiguousarray(self.sym_idx if self.sym_idx.size else np.zeros(1, np.uint32),
                                  dtype=np.uint32)
        args = (self.n_meas, self.row_ptr.ctypes.data, si.ctypes.data, len(detectors),
                det_ptr.ctypes.data, det_meas.ctypes.data, rp.ctypes.data)
        N.check(L.sp_detector_rows(*args, None, 0, C.byref(nnz)))
        out = np.zeros(max(nnz.value, 1), dtype=np.uint32)
        N.check(L.sp_detector_rows(*args, out.ctypes.data, out.size, C.byref(nnz)))
        return InitResult(self.n_qubits, self.n_sym, rp, out[:nnz.value], self.groups)

    def dense_words(self) -> np.ndarray:
        """M_sym as dense row-major u64 words [n_meas][ceil(n_sym/64)]."""
        ldm = max((self.n_sym + 63) // 64, 1)
        W = np.zeros((self.n_meas, ldm), dtype=np.uint64)
        rows = np.repeat(np.arange(self.n_meas), np.diff(self.row_ptr).astype(np.int64))
        s = self.sym_idx.astype(np.uint64)
        np.bitwise_xor.at(W, (rows, (s // 64).astype(np.int64)), np.uint64(1) << (s % 64))
        return W


def run_initialization(text: str) -> InitResult:
    """parse_circuit + run_initialization in the native host front end."""
    L = N.lib()
    m = C.c_void_p()
    N.check(L.sp_model_from_text(text.encode(), C.byref(m)))
    try:
        d = [C.c_uint64() for _ in range(5)]
        N.check(L.sp_model_dims(m, *[C.byref(x) for x in d]))
        nq, nm, ns, ng, nnz = (x.value for x in d)
        row_ptr = np.zeros(nm + 1, dtype=np.uint64)
        sym_idx = np.zeros(max(nnz, 1), dtype=np.uint32)
        groups = np.zeros(ng, dtype=GROUP_DTYPE)
        N.check(L.sp_model_export(m, row_ptr.ctypes.data, sym_idx.ctypes.data, groups.ctypes.data))
        return InitResult(nq, ns, row_ptr, sym_idx[:nnz], groups)
    finally:
        L.sp_model_destroy(m)


parse_and_initialize = run_initialization


def words(n_shots: int) -> int:
    return (n_shots + 63) // 64


class Sampler:
    """One device context (sp_ctx) with a loaded M_sym + channel table."""

    def __init__(self, init: InitResult | None = None, device: int = 0, rng: str = "philox",
                 stream=None):
        import torch

        self._torch = torch
        self.device = device
        L = N.lib()
        self._L = L
        h = C.c_void_p()
        N.check(L.sp_ctx_create(device, C.byref(h)))
        self._h = h
        if stream is not None:
            self.set_stream(stream)
        self.set_rng(rng)
        self.n_meas = self.n_sym = None
        if init is not None:
            self.load(init)

    def close(self):
        if getattr(self, "_h", None):
            self._L.sp_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- configuration ------------------------------------------------------
    def set_stream(self, stream):
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        N.check(self._L.sp_set_stream(self._h, C.c_void_p(handle)))

    def set_rng(self, rng: str):
        N.check(self._L.sp_set_rng(self._h, RNGS[rng]))

    def set_product(self, variant: str):
        N.check(self._L.sp_set_product(self._h, PRODUCTS[variant]))

    def load(self, init: InitResult):
        self.load_csr(init.row_ptr, init.sym_idx, init.n_sym)
        self.load_groups(init.groups)

    def load_csr(self, row_ptr, sym_idx, n_sym: int):
        rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        si = np.ascontiguousarray(sym_idx, dtype=np.uint32)
        if si.size == 0:
            si = np.zeros(1, dtype=np.uint32)
        N.check(self._L.sp_load_msym_csr(self._h, len(rp) - 1, n_sym, rp.ctypes.data,
                                         si.ctypes.data))
        self.n_meas, self.n_sym = len(rp) - 1, n_sym

    def load_dense(self, words_: np.ndarray, n_sym: int):
        w = np.ascontiguousarray(words_, dtype=np.uint64)
        N.check(self._L.sp_load_msym_dense(self._h, w.shape[0], n_sym, w.ctypes.data, w.shape[1]))
        self.n_meas, self.n_sym = w.shape[0], n_sym

    def load_groups(self, groups: np.ndarray):
        g = np.ascontiguousarray(groups, dtype=GROUP_DTYPE)
        N.check(self._L.sp_load_groups(self._h, len(g), g.ctypes.data))

    @property
    def shot_tile(self) -> int:
        t = C.c_uint64()
        N.check(self._L.sp_shot_tile(self._h, C.byref(t)))
        return t.value

    PLAN_FIELDS = ("shot_tile", "gen_warps", "cta_threads", "staged", "row_staged", "lp",
                   "pad_pred", "n_paths", "n_rounds", "n_keep", "n_segments", "n_classes",
                   "n_dense", "nnz_d", "smem_bytes", "fused_ok")

    def plan_info(self) -> dict:
        """Launch shape / table sizes the planner chose for the fused sampler."""
        buf = (C.c_uint64 * 16)()
        N.check(self._L.sp_plan_info(self._h, C.cast(buf, C.c_void_p)))
        return dict(zip(self.PLAN_FIELDS, (int(x) for x in buf)))

    SAMPLER_KERNELS = {0: "d_segments + k2 product", 1: "k1_fused", 2: "k5_columns", 3: "k7_queued"}

    def sampler_kernel(self, tiled: bool = False, detector_counts: bool = False) -> str:
        """Kernel that serves one kind of sample / sample_tiled / sample_counted
        launch (the launch autotune picks K1 or its queued form K7 per kind)."""
        v = C.c_uint32()
        N.check(self._L.sp_sampler_kernel(self._h, int(tiled), int(detector_counts), C.byref(v)))
        return self.SAMPLER_KERNELS[int(v.value)]

    @property
    def launches(self) -> int:
        return int(self._L.sp_launch_count(self._h))

    def synchronize(self):
        N.check(self._L.sp_synchronize(self._h))

    # -- allocation helpers ---------------------------------------------------
    def empty_bits(self, rows: int, n_shots: int):
        return self._torch.empty((rows, max(words(n_shots), 1)), dtype=self._torch.int64,
                                 device=f"cuda:{self.device}")

    def _check_dev(self, t, min_words: int, what: str):
        """The C ABI takes raw device pointers and cannot see buffer sizes:
        check dtype, device and size here before any device write."""
        if t is None:
            return
        if t.dtype != self._torch.int64 and t.dtype != self._torch.uint64:
            raise TypeError(f"{what}: expected int64/uint64 words, got {t.dtype}")
        if t.device.type != "cuda" or t.device.index != self.device:
            raise ValueError(f"{what}: expected a tensor on cuda:{self.device}, got {t.device}")
        if not t.is_contiguous():
            raise ValueError(f"{what}: must be contiguous")
        if t.numel() < min_words:
            raise ValueError(f"{what}: needs >= {min_words} words, has {t.numel()}")

    def _check_matrix(self, t, rows: int, n_shots: int, what: str):
        self._check_dev(t, 0, what)
        if t.dim() != 2 or t.shape[0] < rows or t.shape[1] < words(n_shots):
            raise ValueError(f"{what}: needs shape >= ({rows}, {words(n_shots)}), "
                             f"got {tuple(t.shape)}")

    # -- hot path -------------------------------------------------------------
    def sample(self, n_shots: int, seed: int, shot_begin: int = 0, out=None, counts=None):
        """Fused draw_assignments + sample (K1/K4): measurement-major records."""
        if out is None:
            out = self.empty_bits(self.n_meas, n_shots)
        self._check_matrix(out, self.n_meas, n_shots, "out")
        self._check_dev(counts, self.n_meas, "counts")
        N.check(self._L.sp_sample(self._h, seed, shot_begin, n_shots, _ptr(out), out.shape[1],
                                  _ptr(counts)))
        return out

    def tiled_words(self, n_shots: int) -> int:
        """u64 words of the tiled record array for n_shots."""
        return int(self._L.sp_tiled_words(self._h, n_shots))

    def sample_tiled(self, n_shots: int, seed: int, shot_begin: int = 0, out=None, counts=None):
        """Fused sampler with tiled records: blocks [n_meas][T/64] per T shots."""
        if out is None:
            out = self._torch.empty(max(self.tiled_words(n_shots), 1), dtype=self._torch.int64,
                                    device=f"cuda:{self.device}")
        self._check_dev(out, self.tiled_words(n_shots), "out")
        self._check_dev(counts, self.n_meas, "counts")
        N.check(self._L.sp_sample_tiled(self._h, seed, shot_begin, n_shots, _ptr(out),
                                        _ptr(counts)))
        return out

    def set_detectors(self, detectors):
        """Registers detectors (lists of measurement indices) whose flip counts
        sample_counted() accumulates in the sampling launch."""
        import ctypes as C
        import numpy as np
        ptr = np.zeros(len(detectors) + 1, dtype=np.uint64)
        for i, d in enumerate(detectors):
            ptr[i + 1] = ptr[i] + len(d)
        meas = np.fromiter((m for d in detectors for m in d), dtype=np.uint32, count=int(ptr[-1]))
        self._det_arrays = (ptr, meas)
        N.check(self._L.sp_set_detectors(self._h, len(detectors),
                                         ptr.ctypes.data_as(C.c_void_p),
                                         meas.ctypes.data_as(C.c_void_p) if meas.size else None))
        self.n_det = len(detectors)

    def sample_counted(self, n_shots: int, seed: int, shot_begin: int = 0, out=None, counts=None,
                       det_counts=None, tiled: bool = False):
        """sample / sample_tiled plus per-detector counts (sp_sample_ex):
        det_counts[k] += number of shots in which detector k is 1."""
        if out is None:
            out = (self._torch.empty(max(self.tiled_words(n_shots), 1), dtype=self._torch.int64,
                                     device=f"cuda:{self.device}") if tiled
                   else self.empty_bits(self.n_meas, n_shots))
        if tiled:
            self._check_dev(out, self.tiled_words(n_shots), "out")
            ld = 0
        else:
            self._check_matrix(out, self.n_meas, n_shots, "out")
            ld = out.shape[1]
        self._check_dev(counts, self.n_meas, "counts")
        self._check_dev(det_counts, getattr(self, "n_det", 0), "det_counts")
        N.check(self._L.sp_sample_ex(self._h, seed, shot_begin, n_shots, _ptr(out), ld,
                                     _ptr(counts), _ptr(det_counts)))
        return out

    def untile(self, tiled, n_shots: int, out=None):
        """Tiled records -> measurement-major words [n_meas, ceil(n/64)]."""
        if out is None:
            out = self.empty_bits(self.n_meas, n_shots)
        self._check_dev(tiled, self.tiled_words(n_shots), "tiled")
        self._check_matrix(out, self.n_meas, n_shots, "out")
        N.check(self._L.sp_untile(self._h, _ptr(tiled), n_shots, _ptr(out), out.shape[1]))
        return out

    def encode_tiled(self, tiled, n_shots: int, fmt: str = "b8", out=None):
        size = self.encoded_size(n_shots, fmt)
        if out is None:
            out = self._torch.empty(max(size, 1), dtype=self._torch.uint8,
                                    device=f"cuda:{self.device}")
        N.check(self._L.sp_encode_tiled(self._h, _ptr(tiled), n_shots, FORMATS[fmt], _ptr(out)))
        return out[:size]

    def draw_assignments(self, n_shots: int, seed: int, shot_begin: int = 0, out=None):
        """draw_assignments: the symbol assignment matrix S (row 0 = ones)."""
        if out is None:
            out = self.empty_bits(self.n_sym, n_shots)
        self._check_matrix(out, self.n_sym, n_shots, "out")
        N.check(self._L.sp_draw_assignments(self._h, seed, shot_begin, n_shots, _ptr(out),
                                            out.shape[1]))
        return out

    def sample_given(self, S, n_shots: int, n_sym_S: int | None = None, out=None):
        """sample(expressions, batch) on a supplied bit-sliced S (K2)."""
        n_sym_S = S.shape[0] if n_sym_S is None else n_sym_S
        if out is None:
            out = self.empty_bits(self.n_meas, n_shots)
        self._check_matrix(S, n_sym_S, n_shots, "S")
        self._check_matrix(out, self.n_meas, n_shots, "out")
        N.check(self._L.sp_sample_given_S(self._h, _ptr(S), n_sym_S, S.shape[1], n_shots,
                                          _ptr(out), out.shape[1]))
        return out

    def encode(self, m, n_shots: int, fmt: str = "b8", n_meas: int | None = None, out=None):
        """encode_shots (K3) into a device byte buffer."""
        n_meas = m.shape[0] if n_meas is None else n_meas
        size = int(self._L.sp_encoded_size(n_meas, n_shots, FORMATS[fmt]))
        if out is None:
            out = self._torch.empty(max(size, 1), dtype=self._torch.uint8,
                                    device=f"cuda:{self.device}")
        N.check(self._L.sp_encode(self._h, _ptr(m), m.shape[1], n_meas, n_shots, FORMATS[fmt],
                                  _ptr(out)))
        return out[:size]

    def encoded_size(self, n_shots: int, fmt: str = "b8") -> int:
        return int(self._L.sp_encoded_size(self.n_meas, n_shots, FORMATS[fmt]))

    def sample_to_host(self, n_shots: int, seed: int, fmt: str = "b8", shot_begin: int = 0,
                       out=None):
        """cmd_sample's timed region into a host buffer (numpy or pinned torch)."""
        size = self.encoded_size(n_shots, fmt)
        if out is None:
            out = np.empty(max(size, 1), dtype=np.uint8)
        cap = out.numel() if hasattr(out, "numel") else out.nbytes
        written = C.c_uint64()
        N.check(self._L.sp_sample_to_host(self._h, seed, shot_begin, n_shots, FORMATS[fmt],
                                          _ptr(out), cap, C.byref(written)))
        return out, written.value

    def debug_philox(self, ctr, key):
        a = (C.c_uint32 * 6)(*ctr, *key)
        o = (C.c_uint32 * 4)()
        N.check(self._L.sp_debug_philox(self._h, C.cast(a, C.c_void_p), C.cast(o, C.c_void_p)))
        return list(o)


def unpack_bits(words_: np.ndarray, n_cols: int) -> np.ndarray:
    """Bit-sliced u64 words [rows, ld] -> uint8 0/1 matrix [rows, n_cols]."""
    w = np.ascontiguousarray(words_).view(np.uint8)
    bits = np.unpackbits(w.reshape(words_.shape[0], -1), axis=1, bitorder="little")
    return bits[:, :n_cols]


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """uint8 0/1 matrix [rows, n_cols] -> bit-sliced u64 words [rows, ceil(n/64)]."""
    rows, n = bits.shape
    ld = max((n + 63) // 64, 1)
    pad = np.zeros((rows, ld * 64), dtype=np.uint8)
    pad[:, :n] = bits
    return np.packbits(pad, axis=1, bitorder="little").view(np.uint64).reshape(rows, ld)
