"""ctypes binding of the C ABI declared in include/ffconv_he.h.

This is the whole host<->device boundary: plain pointers, sizes and opaque
handles.  `load_library(path)` binds every symbol of the header to a shared
object; the product loads the CUDA build (`libffconv_he.so`, see
`paper_2102_03494_b200/build.py`) and raises if it is missing.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p

import numpy as np

FHE_MAX_Q = 24
FHE_MAX_P = 2
FHE_MAX_B = 26
FHE_MAX_T = 8

PACKAGE_DIR = os.path.dirname(os.path.abspath(__file__))
# FFCONV_HE_LIB: an alternative in-tree build of the same library (experiment variants)
CUDA_LIB_PATH = os.environ.get("FFCONV_HE_LIB") or os.path.join(PACKAGE_DIR, "_lib", "libffconv_he.so")


class FheParams(ctypes.Structure):
    _fields_ = [
        ("log_n", c_uint32),
        ("L", c_uint32),
        ("K", c_uint32),
        ("n_aux", c_uint32),
        ("T", c_uint32),
        ("flags", c_uint32),
        ("q", c_uint64 * FHE_MAX_Q),
        ("p", c_uint64 * FHE_MAX_P),
        ("b", c_uint64 * FHE_MAX_B),
        ("t", c_uint64 * FHE_MAX_T),
        ("seed", c_uint64),
        ("device", c_int32),
        ("reserved", c_int32),
    ]


# every exported symbol: name -> (restype, argtypes)
_U64P = POINTER(c_uint64)
_VPP = POINTER(c_void_p)
SIGNATURES = {
    "fhe_last_error": (c_char_p, []),
    "fhe_backend_name": (c_char_p, []),
    "fhe_ctx_create": (c_int, [POINTER(FheParams), POINTER(c_void_p)]),
    "fhe_ctx_destroy": (None, [c_void_p]),
    "fhe_sync": (c_int, [c_void_p]),
    "fhe_ctx_key_bytes": (c_int, [c_void_p, _U64P]),
    "fhe_keygen_rotations": (c_int, [c_void_p, POINTER(c_uint32), c_uint32]),
    "fhe_ctx_stream": (c_int, [c_void_p, POINTER(c_void_p)]),
    "fhe_peak_modmul": (c_int, [c_void_p, c_uint32, POINTER(c_double)]),
    "fhe_peak_modmul_kind": (c_int, [c_void_p, c_uint32, c_int, POINTER(c_double)]),
    "fhe_work_modmuls": (c_int, [c_void_p, POINTER(c_double)]),
    "fhe_prof_enable": (c_int, [c_void_p, c_int]),
    "fhe_prof_report": (c_int, [c_void_p, ctypes.c_char_p, c_uint32]),
    "fhe_launch_count": (c_int, [c_void_p, _U64P]),
    "fhe_ct_create": (c_int, [c_void_p, c_uint32, c_uint32, POINTER(c_void_p)]),
    "fhe_ct_destroy": (None, [c_void_p]),
    "fhe_ct_level": (c_uint32, [c_void_p]),
    "fhe_ct_rows": (c_uint32, [c_void_p]),
    "fhe_ct_read": (c_int, [c_void_p, c_void_p, _U64P]),
    "fhe_ct_write": (c_int, [c_void_p, c_void_p, _U64P]),
    "fhe_ct_zero": (c_int, [c_void_p, c_void_p]),
    "fhe_ct_to_device": (c_int, [c_void_p, c_void_p, c_void_p]),
    "fhe_ct_from_device": (c_int, [c_void_p, c_void_p, c_void_p]),
    "fhe_ct_copy": (c_int, [c_void_p, c_void_p, c_void_p]),
    "fhe_capture_begin": (c_int, [c_void_p, c_uint64]),
    "fhe_capture_end": (c_int, [c_void_p, POINTER(c_void_p)]),
    "fhe_graph_launch": (c_int, [c_void_p, c_void_p]),
    "fhe_graph_nodes": (c_int, [c_void_p, _U64P]),
    "fhe_graph_destroy": (None, [c_void_p]),
    "fhe_ctx_peak_bytes": (c_int, [c_void_p, _U64P, c_int]),
    "fhe_pt_create": (c_int, [c_void_p, POINTER(c_void_p)]),
    "fhe_pt_destroy": (None, [c_void_p]),
    "fhe_encode": (c_int, [c_void_p, _U64P, c_void_p]),
    "fhe_pt_read": (c_int, [c_void_p, c_void_p, _U64P]),
    "fhe_encrypt": (c_int, [c_void_p, _U64P, c_uint32, c_void_p]),
    "fhe_decrypt": (c_int, [c_void_p, c_void_p, _U64P]),
    "fhe_decrypt_raw": (c_int, [c_void_p, c_void_p, _U64P]),
    "fhe_check_zero_tail": (c_int, [c_void_p, c_void_p, c_uint32]),
    "fhe_decrypt_slots": (c_int, [c_void_p, c_void_p, c_uint32, c_uint32, _U64P]),
    "fhe_status": (c_int, [c_void_p, POINTER(c_uint32), POINTER(c_uint32), c_int]),
    "fhe_add": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "fhe_mul_plain": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "fhe_mul_plain_acc": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "fhe_mul_scalar": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "fhe_add_plain": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "fhe_rotate": (c_int, [c_void_p, c_void_p, c_uint32, c_void_p]),
    "fhe_mod_switch": (c_int, [c_void_p, c_void_p, c_void_p]),
    "fhe_square": (c_int, [c_void_p, c_void_p, c_void_p]),
    "fhe_rotate_many": (c_int, [c_void_p, _VPP, _VPP, c_uint32, c_uint32]),
    "fhe_rotate_multi": (c_int, [c_void_p, _VPP, _VPP, POINTER(c_uint32), c_uint32]),
    "fhe_rotate_hoisted": (c_int, [c_void_p, c_void_p, POINTER(c_uint32), c_uint32, _VPP]),
    "fhe_rotate_add_many": (c_int, [c_void_p, _VPP, _VPP, c_uint32, c_uint32]),
    "fhe_mul_plain_many": (c_int, [c_void_p, _VPP, _VPP, _VPP, c_uint32]),
    "fhe_hoisted_dot": (c_int, [c_void_p, _VPP, POINTER(c_uint32), c_uint32, _VPP, c_uint32, _VPP]),
    "fhe_add_many": (c_int, [c_void_p, _VPP, _VPP, _VPP, c_uint32]),
    "fhe_rotate_and_sum": (c_int, [c_void_p, _VPP, _VPP, c_uint32, c_uint32]),
    "fhe_combine": (c_int, [c_void_p, _VPP, POINTER(c_uint32), c_uint32, c_void_p]),
    "fhe_ct_gemm": (c_int, [c_void_p, _VPP, c_uint32, POINTER(c_int64), c_uint32, _VPP]),
    "fhe_debug_rotate_stages": (c_int, [c_void_p, c_void_p, c_uint32, _U64P, _U64P, _U64P]),
}


class FheError(RuntimeError):
    """A negative status returned across the C ABI."""


class Library:
    """One loaded implementation of the ABI."""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"evaluator library {path} is missing; build it with "
                f"`python -m paper_2102_03494_b200.build`")
        self.path = path
        self.dll = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(self.dll, name)
            fn.restype = res
            fn.argtypes = args
        self.backend = self.dll.fhe_backend_name().decode()

    def check(self, rc: int, what: str) -> None:
        if rc != 0:
            msg = self.dll.fhe_last_error().decode(errors="replace")
            raise FheError(f"{what} failed ({rc}): {msg}")

    def call(self, name: str, *args):
        rc = getattr(self.dll, name)(*args)
        self.check(rc, name)
        return rc


_CUDA_LIB: Library | None = None


def cuda_library() -> Library:
    """The sm_100a CUDA implementation.  Raises if it was not built."""
    global _CUDA_LIB
    if _CUDA_LIB is None:
        _CUDA_LIB = Library(CUDA_LIB_PATH)
        if _CUDA_LIB.backend != "cuda-sm100a":
            raise FheError(f"{CUDA_LIB_PATH} reports backend {_CUDA_LIB.backend!r}")
    return _CUDA_LIB


def u64_ptr(arr: np.ndarray):
    assert arr.dtype == np.uint64 and arr.flags["C_CONTIGUOUS"]
    return arr.ctypes.data_as(_U64P)


def handle_array(handles) -> ctypes.Array:
    arr = (c_void_p * len(handles))()
    for i, h in enumerate(handles):
        arr[i] = h
    return arr
