"""ctypes binding of the C ABI in ``include/approx8_b200.h``.

The library is the product: there is no Python/NumPy/torch fallback for any
compute path.  If ``_lib/libapprox8_b200.so`` is missing this module raises
at import (build it with ``python paper_1511_04561_b200/build.py``).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import ConfigError, InputError, UsageError

_LIB_PATH = Path(os.environ.get("A8_LIB") or Path(__file__).resolve().parent / "_lib" / "libapprox8_b200.so")

A8_OK, A8_ERR_INPUT, A8_ERR_CONFIG, A8_ERR_USAGE, A8_ERR_CUDA = 0, 1, 2, 3, 4
A8_STATUS_NONFINITE = 1
A8_STATUS_AMAX_MISMATCH = 2
A8_PRODUCE_SCALE, A8_PRODUCE_RELU, A8_PRODUCE_RELU_MASK = 0, 1, 2
A8_LAYOUT_STATUS_COUNT = 1
KIND_CODE = {"dynamic-tree": 0, "static-tree": 1, "linear": 2, "mantissa": 3}
NORM_CODE = {"none": 0, "absmax": 1, "decade": 2}
LUT_MAX = 4096


class Book(C.Structure):
    _fields_ = [
        ("values", C.c_double * 128),
        ("table", C.c_float * 256),
        ("codes", C.c_uint8 * 128),
        ("ndistinct", C.c_int32),
        ("kind", C.c_int32),
        ("pad", C.c_int32 * 2),
    ]


class Lut(C.Structure):
    _fields_ = [
        ("len", C.c_uint32),
        ("kbase", C.c_int32),
        ("valid", C.c_uint32),
        ("nfinite", C.c_uint32),
        ("scale", C.c_float),
        ("pad", C.c_uint32 * 3),
        ("T", C.c_uint32 * 128),
        ("e", C.c_uint32 * LUT_MAX),
    ]


class EncSeg(C.Structure):
    _fields_ = [
        ("x", C.c_void_p),
        ("n", C.c_int64),
        ("flat_off", C.c_int64),
        ("scale_idx", C.c_int32),
        ("pad", C.c_int32),
    ]


class EncSeg64(C.Structure):
    _fields_ = [
        ("x", C.c_void_p),
        ("n", C.c_int64),
        ("flat_off", C.c_int64),
        ("scale_idx", C.c_int32),
        ("pad", C.c_int32),
    ]


class DecSeg(C.Structure):
    _fields_ = [
        ("out", C.c_void_p),
        ("n", C.c_int64),
        ("flat_off", C.c_int64),
        ("scale_idx", C.c_int32),
        ("pad", C.c_int32),
    ]


class ProdSeg(C.Structure):
    _fields_ = [("x", C.c_void_p), ("y", C.c_void_p), ("mask", C.c_void_p), ("n", C.c_int64)]


class ObQSeg(C.Structure):
    _fields_ = [("g", C.c_void_p), ("residual", C.c_void_p), ("n", C.c_int64), ("bits", C.c_void_p),
                ("levels", C.c_void_p), ("status", C.c_void_p)]


class ObSeg(C.Structure):
    _fields_ = [("out", C.c_void_p), ("n", C.c_int64), ("bit_off", C.c_int64)]


class Layout(C.Structure):
    _fields_ = [
        ("codes", C.c_void_p),
        ("scales", C.c_void_p),
        ("block_len", C.c_int64),
        ("block_stride", C.c_int64),
        ("scale_block_stride", C.c_int64),
        ("rank_stride", C.c_int64),
        ("scale_reps", C.c_int32),
        ("flags", C.c_int32),
    ]


# every symbol include/approx8_b200.h declares, with its ctypes signature
SIGNATURES = {
    "a8_abi_version": (C.c_int, []),
    "a8_last_error": (C.c_char_p, []),
    "a8_codebook": (C.c_int, [C.c_int, C.POINTER(Book)]),
    "a8_fixed_scale": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "a8_build_lut_host": (C.c_int, [C.POINTER(Book), C.c_float, C.POINTER(Lut)]),
    "a8_workspace_bytes": (C.c_size_t, [C.c_int]),
    "a8_encode": (
        C.c_int,
        [C.POINTER(EncSeg), C.c_int, C.c_void_p, C.c_int, C.c_void_p, Layout, C.c_void_p,
         C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p],
    ),
    "a8_encode_premax": (
        C.c_int,
        [C.POINTER(EncSeg), C.c_int, C.c_void_p, C.c_void_p, Layout, C.c_void_p, C.c_size_t, C.c_void_p,
         C.c_void_p, C.c_void_p],
    ),
    "a8_produce_absmax": (C.c_int, [C.POINTER(ProdSeg), C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_void_p]),
    "a8_encode_f64": (
        C.c_int,
        [C.POINTER(EncSeg64), C.c_int, C.c_void_p, C.c_int, C.c_float, Layout, C.c_void_p, C.c_size_t,
         C.c_void_p, C.c_void_p, C.c_void_p],
    ),
    "a8_decode": (
        C.c_int,
        [C.POINTER(DecSeg), C.c_int, C.c_void_p, Layout, C.c_int, C.c_int, C.c_int, C.c_int,
         C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p],
    ),
    "a8_decode_peers": (C.c_int, [C.POINTER(DecSeg), C.c_int, C.c_void_p, Layout, C.POINTER(C.c_void_p), C.c_int,
                                  C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "a8_decode_local": (
        C.c_int,
        [C.POINTER(DecSeg), C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_void_p, Layout, C.c_int, C.c_int, C.c_int,
         C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p],
    ),
    "a8_encode_trace": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_uint64)]),
    "a8_onebit_workspace_bytes": (C.c_size_t, []),
    "a8_onebit_quantize": (
        C.c_int,
        [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
         C.c_size_t, C.c_void_p],
    ),
    "a8_onebit_multi_workspace_bytes": (C.c_size_t, [C.c_int]),
    "a8_onebit_quantize_multi": (C.c_int, [C.POINTER(ObQSeg), C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]),
    "a8_onebit_decode": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "a8_onebit_reduce": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                   C.c_int, C.c_void_p, C.c_void_p]),
    "a8_roundtrip": (
        C.c_int,
        [C.POINTER(EncSeg), C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
         C.c_void_p, C.c_size_t, C.c_void_p],
    ),
    "a8_encode_blocked": (
        C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
    ),
    "a8_decode_blocked": (
        C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
    ),
    "a8_error_workspace_bytes": (C.c_size_t, []),
    "a8_error_stats": (
        C.c_int,
        [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
         C.c_void_p, C.c_size_t, C.c_void_p],
    ),
    "a8_device_info": (
        C.c_int,
        [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
    ),
}


def _load() -> C.CDLL:
    if not _LIB_PATH.exists():
        raise ImportError(
            f"approx8 B200 library not built: {_LIB_PATH} is missing. "
            "Run `python paper_1511_04561_b200/build.py` (needs nvcc); there is no CPU fallback."
        )
    lib = C.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_LOCAL", 0))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.a8_abi_version() != 1:
        raise ImportError("approx8 B200 library ABI mismatch; rebuild it")
    return lib


lib = _load()
LIB_PATH = _LIB_PATH


def check(rc: int) -> None:
    """Map a C status to the reference's exception taxonomy (errors.py:16-33)."""
    if rc == A8_OK:
        return
    msg = (lib.a8_last_error() or b"").decode(errors="replace")
    if rc == A8_ERR_INPUT:
        raise InputError(msg)
    if rc == A8_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == A8_ERR_USAGE:
        raise UsageError(msg)
    raise RuntimeError(f"approx8 CUDA failure: {msg}")


def workspace_bytes(nseg: int) -> int:
    return int(lib.a8_workspace_bytes(int(nseg)))
