"""ctypes binding of ``librmgpu.so`` (the C-ABI in ``include/rmgpu.h``).

The library is loaded from this package directory only (in-tree build). There is no CPU
fallback: if the library or a CUDA device is missing, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RMGPU_LIB_PATH") or os.path.join(_PKG, "librmgpu.so")  # override: tuning experiments
HOSTLIB_PATH = os.path.join(_PKG, "librectmorph_b200.so")

_P, _S, _I, _U, _U64 = C.c_void_p, C.c_size_t, C.c_int, C.c_uint, C.c_uint64

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "rmgpu_morph_u8": [_P, _S, _P, _S, _I, _I, _I, _I, _I, _I, _U, _I, _I, _P],
    "rmgpu_morph_u16": [_P, _S, _P, _S, _I, _I, _I, _I, _I, _I, _U, _I, _I, _P],
    "rmgpu_morph_batched_u8": [_P, _S, _S, _P, _S, _S, _I, _I, _I, _I, _I, _I, _I, _U, _P],
    "rmgpu_morph_batched_u16": [_P, _S, _S, _P, _S, _S, _I, _I, _I, _I, _I, _I, _I, _U, _P],
    "rmgpu_morph_band_u8": [_P, _S, _P, _S, _I, _I, _I, _I, _I, _I, _I, _I, _U, _P],
    "rmgpu_morph_band_u16": [_P, _S, _P, _S, _I, _I, _I, _I, _I, _I, _I, _I, _U, _P],
    "rmgpu_pass_u8": [_I, _P, _S, _P, _S, _I, _I, _I, _I, _I, _U, _I, _P],
    "rmgpu_window_1d_u8": [_P, _S, _I, _I, _I, _U, _I, _P, _P],
    "rmgpu_transpose_u8": [_P, _S, _P, _S, _I, _I, _P],
    "rmgpu_transpose_u16": [_P, _S, _P, _S, _I, _I, _P],
    "rmgpu_transpose_tiles_u8": [_P, _S, _I, _S, _S, _P],
    "rmgpu_transpose_tiles_u16": [_P, _S, _I, _S, _S, _P],
    "rmgpu_transpose_tiles_u32": [_P, _S, _I, _S, _S, _P],
    "rmgpu_morph_host_u8": [_P, _S, _P, _S, _I, _I, _I, _I, _I, _I, _U, _I, _I],
    "rmgpu_morph_host_u16": [_P, _S, _P, _S, _I, _I, _I, _I, _I, _I, _U, _I, _I],
    "rmgpu_transpose_host_u8": [_P, _S, _P, _S, _I, _I],
    "rmgpu_transpose_host_u16": [_P, _S, _P, _S, _I, _I],
    "rmgpu_transpose_tiles_host": [_P, _I, _S, _I, _S, _S],
    "rmgpu_pass_host_u8": [_I, _P, _S, _P, _S, _I, _I, _I, _I, _I, _U, _I],
    "rmgpu_window_1d_host_u8": [_P, _S, _I, _I, _I, _U, _I, _P],
    "rmgpu_resolve": [_I, _I, _I, _I, _I],
    "rmgpu_format_config": [_I, _I, _I, C.c_char_p, _S],
    "rmgpu_parse_config": [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "rmgpu_calibrate": [_I, _I, C.POINTER(C.c_int), _I, _I, C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "rmgpu_generate_u8": [_P, _S, _I, _I, _U64, _U64, _P],
    "rmgpu_generate_u16": [_P, _S, _I, _I, _U64, _U64, _P],
    "rmgpu_abi_version": [],
    "rmgpu_last_error": [],
    "rmgpu_status_string": [_I],
    "rmgpu_launch_count": [],
    "rmgpu_plan_name": [_I, _I, _I, _I, _I, _I],
    "rmgpu_debug_trace": [_P, _I],
    "rmgpu_debug_set": [C.c_char_p, _I],
}
_RESTYPES = {
    "rmgpu_last_error": C.c_char_p,
    "rmgpu_status_string": C.c_char_p,
    "rmgpu_launch_count": C.c_ulonglong,
    "rmgpu_plan_name": C.c_char_p,
    "rmgpu_debug_trace": None,
    "rmgpu_debug_set": None,
}

_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    """Load librmgpu.so from the package directory (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2002_09474_b200.build` "
                    "(there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, args in SIGNATURES.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = _RESTYPES.get(name, C.c_int)
            _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
