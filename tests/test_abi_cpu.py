"""The C-ABI library loads and exports every symbol include/*.h declares; host
entry points behave on a machine without a GPU."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2311_03906_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in re.finditer(r"^\s*[A-Za-z_][\w\s\*]*?\b(sp_\w+)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return names


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("sp_sample", "sp_sample_given_S", "sp_draw_assignments", "sp_encode",
                 "sp_load_msym_csr", "sp_load_msym_dense", "sp_load_groups", "sp_set_rng",
                 "sp_ctx_create", "sp_ctx_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    bound = {n for n, _, _ in _native.SIGNATURES}
    assert declared_functions() == bound


def test_abi_version_and_group_struct():
    assert _native.lib().sp_abi_version() == 1
    assert C.sizeof(_native.sp_group) == 24


def test_ctx_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = _native.lib().sp_ctx_create(0, C.byref(h))
    assert rc == -5  # SP_ERR_CUDA
    assert _native.lib().sp_last_error()


def test_encoded_size():
    L = _native.lib()
    assert L.sp_encoded_size(3, 1, 0) == 4
    assert L.sp_encoded_size(9, 5, 1) == 10
    assert L.sp_encoded_size(145, 10, 1) == 190


def test_error_mapping():
    with pytest.raises(_native.InvalidArgument):
        _native.check(-1)
    with pytest.raises(IndexError):
        _native.check(-2)
