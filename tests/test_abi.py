"""The C-ABI boundary: every symbol declared in include/ffconv_he.h is exported by
both implementations (CUDA build and golden model) and bound by abi.py.  Loading
the CUDA library needs no GPU; no compute is called here."""

import ctypes
import os
import re

import pytest

from paper_2102_03494_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    with open(os.path.join(ROOT, "include", "ffconv_he.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(fhe_\w+)\s*\(", text)))


def test_header_fully_bound():
    assert set(header_functions()) == set(abi.SIGNATURES)


def test_cuda_library_exports_every_symbol():
    from paper_2102_03494_b200.build import build
    path = build()
    lib = ctypes.CDLL(path)
    for name in header_functions():
        assert hasattr(lib, name), name
    lib.fhe_backend_name.restype = ctypes.c_char_p
    assert lib.fhe_backend_name() == b"cuda-sm100a"


def test_golden_library_exports_every_symbol(golden_lib):
    for name in header_functions():
        assert hasattr(golden_lib.dll, name), name
    assert golden_lib.backend == "golden-c"


def test_params_struct_layout():
    # 6 u32 + 24+2+26+8 u64 + u64 seed + 2 i32
    assert ctypes.sizeof(abi.FheParams) == 6 * 4 + (24 + 2 + 26 + 8) * 8 + 8 + 8


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(FileNotFoundError):
        abi.Library(str(tmp_path / "nope.so"))
