"""ctypes binding of libsymphase_b200.so (include/symphase_b200.h).

The library is built in-tree by `__graft_entry__.build()` (or
`make -C paper_2311_03906_b200/csrc`). There is no fallback: importing the
sampler without the built library raises, so nothing silently runs on the
CPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("SP_LIB") or Path(__file__).resolve().parent / "libsymphase_b200.so")  # SP_LIB: A/B tools only

SP_OK = 0
STATUS = {
    -1: "SP_ERR_INVALID_ARGUMENT",
    -2: "SP_ERR_OUT_OF_RANGE",
    -3: "SP_ERR_PARSE",
    -4: "SP_ERR_LOGIC",
    -5: "SP_ERR_CUDA",
    -6: "SP_ERR_NOT_LOADED",
    -7: "SP_ERR_UNSUPPORTED",
}


class sp_group(C.Structure):
    _fields_ = [
        ("dist", C.c_uint8),
        ("reserved", C.c_uint8 * 7),
        ("param", C.c_double),
        ("first_symbol", C.c_uint32),
        ("arity", C.c_uint32),
    ]


# (name, restype, argtypes) for every symbol include/symphase_b200.h declares.
_u64, _u32, _i = C.c_uint64, C.c_uint32, C.c_int
_p, _pu64, _pu32 = C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)
SIGNATURES = [
    ("sp_last_error", C.c_char_p, []),
    ("sp_abi_version", _i, []),
    ("sp_model_from_text", _i, [C.c_char_p, C.POINTER(_p)]),
    ("sp_model_destroy", None, [_p]),
    ("sp_parse_circuit", _i, [C.c_char_p, _u64, _p, _p, _p, _p, _u64, _p, _pu64, _pu64]),
    ("sp_model_from_program", _i, [_u64, _p, _p, _p, _p, C.POINTER(_p)]),
    ("sp_model_dims", _i, [_p, _pu64, _pu64, _pu64, _pu64, _pu64]),
    ("sp_model_export", _i, [_p, _p, _p, _p]),
    ("sp_detector_rows", _i, [_u64, _p, _p, _u64, _p, _p, _p, _p, _u64, _pu64]),
    ("sp_ctx_create", _i, [_i, C.POINTER(_p)]),
    ("sp_ctx_destroy", None, [_p]),
    ("sp_set_stream", _i, [_p, _p]),
    ("sp_set_rng", _i, [_p, _i]),
    ("sp_set_product", _i, [_p, _i]),
    ("sp_load_msym_csr", _i, [_p, _u64, _u64, _p, _p]),
    ("sp_load_msym_dense", _i, [_p, _u64, _u64, _p, _u64]),
    ("sp_load_groups", _i, [_p, _u64, _p]),
    ("sp_load_model", _i, [_p, _p]),
    ("sp_shot_tile", _i, [_p, _pu64]),
    ("sp_sample", _i, [_p, _u64, _u64, _u64, _p, _u64, _p]),
    ("sp_draw_assignments", _i, [_p, _u64, _u64, _u64, _p, _u64]),
    ("sp_tiled_words", _u64, [_p, _u64]),
    ("sp_sample_tiled", _i, [_p, _u64, _u64, _u64, _p, _p]),
    ("sp_set_detectors", _i, [_p, _u64, _p, _p]),
    ("sp_sample_ex", _i, [_p, _u64, _u64, _u64, _p, _u64, _p, _p]),
    ("sp_untile", _i, [_p, _p, _u64, _p, _u64]),
    ("sp_encode_tiled", _i, [_p, _p, _u64, _i, _p]),
    ("sp_sample_given_S", _i, [_p, _p, _u64, _u64, _u64, _p, _u64]),
    ("sp_encoded_size", _u64, [_u64, _u64, _i]),
    ("sp_encode", _i, [_p, _p, _u64, _u64, _u64, _i, _p]),
    ("sp_sample_to_host", _i, [_p, _u64, _u64, _u64, _i, _p, _u64, _pu64]),
    ("sp_debug_philox", _i, [_p, _p, _p]),
    ("sp_debug_timers", _i, [_p, _p]),
    ("sp_plan_info", _i, [_p, _p]),
    ("sp_sampler_kernel", _i, [_p, _i, _i, _pu32]),
    ("sp_launch_count", _u64, [_p]),
    ("sp_synchronize", _i, [_p]),
]

_lib = None


def lib() -> C.CDLL:
    """Load the native library, failing loudly when it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH.name} is not built (expected at {LIB_PATH}); run "
                "`python -c 'import __graft_entry__ as g; g.build()'` — there is no CPU fallback")
        L = C.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class SymphaseError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class OutOfRange(SymphaseError, IndexError):
    """std::out_of_range in the reference (sampler.cpp:63-67)."""


class InvalidArgument(SymphaseError, ValueError):
    """std::invalid_argument in the reference (sampler.cpp:50)."""


class ParseError(SymphaseError, ValueError):
    """cliffsym::ParseError (circuit.hpp:42-47)."""


class LogicError(SymphaseError):
    """std::logic_error in the reference (tableau.cpp:138-192)."""


_EXC = {-1: InvalidArgument, -2: OutOfRange, -3: ParseError, -4: LogicError}


def check(code: int) -> None:
    if code != SP_OK:
        msg = lib().sp_last_error().decode(errors="replace")
        raise _EXC.get(code, SymphaseError)(code, msg)
