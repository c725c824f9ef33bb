"""The C-ABI library loads and exports exactly what include/omni.h declares
(CPU-only: no kernel is launched)."""

import ctypes
import os
import re

import pytest

from paper_1606_04487_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "omni.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(?:int|long long|const char\*)\s+(omni_\w+)\s*\(([^)]*)\)\s*;", src):
        args = [a.strip() for a in m.group(2).split(",") if a.strip() and a.strip() != "void"]
        out[m.group(1)] = len(args)
    return out


def test_library_built():
    assert os.path.exists(_abi.LIB_PATH), "run `make` (or __graft_entry__.build()) first"


def test_header_and_binding_agree():
    decl = declared()
    assert len(decl) >= 25
    assert set(decl) == set(_abi.SIGNATURES), set(decl) ^ set(_abi.SIGNATURES)
    for name, n in decl.items():
        assert len(_abi.SIGNATURES[name][1]) == n, (name, n, _abi.SIGNATURES[name][1])


def test_library_exports_every_symbol():
    lib = _abi.load()
    for name in declared():
        assert hasattr(lib, name), name
    assert lib.omni_version() == 1


def test_host_only_entry_points():
    lib = _abi.load()
    # pure host arithmetic: no device needed
    assert lib.omni_pool_out_size(32, 3, 2, 0, 1) == 16
    assert lib.omni_pool_out_size(55, 3, 2, 0, 1) == 27
    assert lib.omni_pool_out_size(5, 7, 1, 0, 1) == -1
    assert lib.omni_bias_grad_ws_elems(10000, 96) > 0


def test_errors_map_to_valueerror_without_gpu():
    # argument validation happens before any CUDA call
    with pytest.raises(ValueError, match="b_p=0 out of range"):
        _abi.call("omni_lower_nchw_f32", None, 2, 1, 8, 3, 1, 1, 0, 0, None, 9, None)
    with pytest.raises(ValueError, match="not divisible by stride"):
        _abi.call("omni_lower_nchw_f32", None, 2, 1, 8, 3, 2, 0, 0, 1, None, 9, None)
    with pytest.raises(ValueError, match="empty problem"):
        _abi.call("omni_gemm_f32", 0, 0, 8, 8, None, 8, 0, None, 8, 0, None, 8, 0, None, None, 0,
                  None, 0, None)
    assert "empty problem" in _abi.last_error()
