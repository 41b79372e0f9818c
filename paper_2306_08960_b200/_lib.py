"""ctypes binding of the C ABI declared in include/bitmm_b200.h.

The product path is the in-tree CUDA library `libbitmm_b200.so`. There is no
CPU fallback: if the library is missing this module raises on load.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG_DIR)
LIB_PATH = os.path.join(PKG_DIR, "libbitmm_b200.so")
HEADER = os.path.join(REPO, "include", "bitmm_b200.h")

OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_INVALID_ENCODING = 2
ERR_CUDA = 3
ERR_NO_DEVICE = 4
ERR_IO = 5

_p = C.c_void_p
_i64 = C.c_int64
_f = C.c_float
_i = C.c_int

# name -> (restype, argtypes); mirrors include/bitmm_b200.h
ROUTINE_1X1, ROUTINE_1X2, ROUTINE_2X2 = 0, 1, 2


class GemmItem(C.Structure):
    """ctypes mirror of `bitmm_gemm_item` (include/bitmm_b200.h); field order and types must
    match the C struct (tests/test_capi_cpu.py compares offsets with gcc's)."""
    _fields_ = [
        ("routine", C.c_int),
        ("a0", _p), ("a1", _p), ("a2", _p),
        ("b0", _p), ("b1", _p), ("b2", _p),
        ("m", _i64), ("n", _i64), ("k", _i64), ("wpr", _i64),
        ("a_scale", _f), ("has_a_gamma", C.c_int), ("a_gamma", _f),
        ("b_scale", _f), ("has_b_gamma", C.c_int), ("b_gamma", _f),
        ("row_scale", _p), ("col_scale", _p),
        ("c_units", _p), ("c", _p), ("ldc", _i64),
    ]


class HostOut(C.Structure):
    """ctypes mirror of `bitmm_host_out` (the late-output callback's destination)."""
    _fields_ = [("c_units", _p), ("c", _p), ("ldc", _i64)]


# int (*bitmm_out_fn)(void* user, bitmm_host_out* out)
OUT_FN = C.CFUNCTYPE(C.c_int, _p, C.POINTER(HostOut))
WANT_UNITS, WANT_C = 1, 2


class BtsrHeader(C.Structure):
    """ctypes mirror of `bitmm_btsr_header`."""
    _fields_ = [("kind", C.c_int), ("rows", _i64), ("cols", _i64), ("words_per_row", _i64),
                ("nnz", _i64)]


SIGNATURES = {
    "bitmm_abi_version": (_i, []),
    "bitmm_last_error": (C.c_char_p, []),
    "bitmm_device_sm_count": (_i, []),
    "bitmm_device_status": (_i, [_p]),
    "bitmm_reserve_workspace": (_i, [C.c_size_t]),
    "bitmm_workspace_bytes": (C.c_size_t, [_i, _i64, _i64, _i64]),
    "bitmm_last_launch_count": (_i, []),
    "bitmm_last_d2h_bytes": (C.c_uint64, []),
    "bitmm_profile_enable": (_i, [_i]),
    "bitmm_profile_collect": (_i, []),
    "bitmm_profile_reset": (_i, []),
    "bitmm_profile_kernel_count": (_i, []),
    "bitmm_profile_kernel_name": (C.c_char_p, [_i]),
    "bitmm_profile_kernel_launches": (_i, [_i]),
    "bitmm_profile_kernel_ms": (C.c_double, [_i]),
    "bitmm_ipc_get_handle": (_i, [_p, _p, C.POINTER(C.c_uint64)]),
    "bitmm_ipc_open": (_i, [_p, C.POINTER(_p)]),
    "bitmm_ipc_close": (_i, [_p]),
    "bitmm_gemm_1x1_dev": (_i, [_p, _i64, _p, _i64, _i64, _i64, _f, _f, _p, _p, _i64, _p]),
    "bitmm_gemm_1x1_host": (_i, [_p, _i64, _p, _i64, _i64, _i64, _f, _f, _p, _p, _i64]),
    "bitmm_gemm_1x1_popc_dev": (_i, [_p, _i64, _p, _i64, _i64, _i64, _f, _f, _p, _p, _i64, _p]),
    "bitmm_gemm_1x2_dev": (
        _i,
        [_p, _i64, _f, _p, _p, _p, _i64, _i64, _i64, _f, _i, _f, _p, _p, _p, _p, _i64, _p],
    ),
    "bitmm_gemm_1x2_host": (
        _i,
        [_p, _i64, _f, _p, _p, _p, _i64, _i64, _i64, _f, _i, _f, _p, _p, _p, _p, _i64],
    ),
    "bitmm_gemm_2x2_dev": (
        _i,
        [_p, _p, _p, _i64, _f, _i, _f, _p, _p, _p, _i64, _i64, _i64, _f, _i, _f, _p, _p, _p, _p,
         _i64, _p],
    ),
    "bitmm_gemm_2x2_host": (
        _i,
        [_p, _p, _p, _i64, _f, _i, _f, _p, _p, _p, _i64, _i64, _i64, _f, _i, _f, _p, _p, _p, _p,
         _i64],
    ),
    "bitmm_gemm_1x32_dev": (_i, [_p, _i64, _i64, _i64, _f, _p, _p, _i64, _i64, _p, _i64, _p]),
    "bitmm_gemm_1x32_host": (_i, [_p, _i64, _i64, _i64, _f, _p, _p, _i64, _i64, _p, _i64]),
    "bitmm_spmm_csr_dev": (_i, [_i64, _i64, _p, _p, _p, _p, _i64, _i64, _p, _i64, _p]),
    "bitmm_spmm_csr_host": (_i, [_i64, _i64, _p, _p, _p, _i64, _p, _i64, _i64, _p, _i64]),
    "bitmm_layer_forward_dev": (
        _i,
        [_i64, _i64, _f, _p, _p, _i64, _p, _p, _p, _p, _i64, _i64, _p, _i64, _p],
    ),
    "bitmm_layer_forward_host": (
        _i,
        [_i64, _i64, _f, _p, _p, _i64, _p, _p, _p, _i64, _p, _i64, _i64, _p, _i64],
    ),
    "bitmm_layer_forward_2bit_dev": (
        _i,
        [_i64, _i64, _f, _p, _p, _i64, _p, _p, _p, _p, _p, _p, _i64, _f, _i, _f, _p, _i64, _p],
    ),
    "bitmm_layer_forward_2bit_host": (
        _i,
        [_i64, _i64, _f, _p, _p, _i64, _p, _p, _p, _i64, _p, _p, _p, _i64, _f, _i, _f, _p, _i64],
    ),
    "bitmm_gemm_batch_dev": (_i, [_p, _i, _p]),
    "bitmm_gemm_host_late": (_i, [_p, _i, _p, _p]),
    "bitmm_gemm_batch_host": (_i, [_p, _i]),
    "bitmm_shard_plan_create": (_i, [_p, _i, _i64, _i64, _i64, _i64, _p]),
    "bitmm_shard_plan_upload": (_i, [_p, _p, _p]),
    "bitmm_shard_run": (_i, [_p, _i, _p]),
    "bitmm_shard_download": (_i, [_p, _i64, _i64, _p, _i64]),
    "bitmm_shard_plan_destroy": (_i, [_p]),
    "bitmm_btsr_read_header": (_i, [C.c_char_p, _p]),
    "bitmm_dot_binary_dev": (_i, [_p, _p, _i64, _i64, _i64, _p, _p]),
    "bitmm_mbm_dev": (_i, [_p, _p, _p, _i64, _i64, _p, _p]),
    "bitmm_dot_binary_host": (_i, [_p, _p, _i64, _i64, _i64, _p]),
    "bitmm_mbm_host": (_i, [_p, _p, _p, _i64, _i64, _p]),
    "bitmm_validate_planes_dev": (_i, [_p, _p, _p, _i64, _i64, _i64, _f, _p]),
    "bitmm_btsr_load_dev": (_i, [C.c_char_p, _i, _p, _p, _p, _p, _p]),
    "bitmm_pack_signs_dev": (_i, [_p, _i64, _i64, _i64, _p, _i64, _p]),
    "bitmm_pack_signs_host": (_i, [_p, _i64, _i64, _i64, _p, _i64]),
    "bitmm_quantize_thm_dev": (_i, [_p, _i64, _i64, _i64, _f, _p, _p, _p, _i64, _p]),
    "bitmm_quantize_thm_host": (_i, [_p, _i64, _i64, _i64, _f, _p, _p, _p, _i64]),
    "bitmm_decompose_thm_dev": (_i, [_p, _i64, _i64, _p, _p, _p, _i64, _p]),
    "bitmm_decompose_thm_host": (_i, [_p, _i64, _i64, _p, _p, _p, _i64]),
    "bitmm_decompose_apb_dev": (_i, [_p, _i64, _i64, _i64, _f, _p, _p, _i64, _p, _p, _p, _i64,
                                     C.POINTER(_i64), _p]),
    "bitmm_decompose_apb_host": (_i, [_p, _i64, _i64, _i64, _f, _p, _p, _i64, _p, _p, _p, _i64,
                                      C.POINTER(_i64)]),
}


class BitmmError(RuntimeError):
    """Raised for BITMM_ERR_CUDA / BITMM_ERR_NO_DEVICE."""


def header_symbols(path: str = HEADER) -> list[str]:
    """Every function name declared in include/bitmm_b200.h."""
    text = open(path).read()
    return sorted(set(re.findall(r"\b(bitmm_[a-z0-9_]+)\s*\(", text)))


_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BitmmError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2306_08960_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().bitmm_last_error().decode(errors="replace")
