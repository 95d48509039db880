"""ctypes binding of the C ABI declared in include/txb.h.

The shared library ``libtxb.so`` is built in-tree by ``build.build_library``
(nvcc, sm_100a SASS, static cudart).  Nothing here falls back to a CPU path:
if the library is missing or fails to load, every product entry point raises
``CudaLaneError``.
"""

from __future__ import annotations

import ctypes
import re
from ctypes import c_char_p, c_int, c_int64, c_void_p, POINTER
from pathlib import Path

from .errors import (CapacityError, CodegenError, ConfigurationError, CudaLaneError, OrientationError,
                     ShapeError)

LIB_PATH = Path(__file__).resolve().parent / "libtxb.so"

TXB_OK, TXB_E_UNSUPPORTED, TXB_E_SHAPE, TXB_E_CONFIG = 0, -1, -2, -3
TXB_E_CAPACITY, TXB_E_ARG, TXB_E_CUDA, TXB_E_ORIENTATION = -4, -5, -6, -7
TXB_E_COMPILE = -8

_I = c_int
_P = c_void_p
# name -> (restype, argtypes); exactly the functions of include/txb.h
SIGNATURES = {
    "txb_abi_version": (_I, []),
    "txb_last_error": (c_char_p, []),
    "txb_query": (_I, [_I, _I, _I, _I, _I, _I]),
    "txb_launch_config": (_I, [_I, _I, _I, _I, _I, _I, c_int64, _I, _I] + [POINTER(c_int)] * 7),
    "txb_integrate_cells": (_I, [_I, _I, _I, _I, _I, _I, _I, c_int64] + [_P] * 8 + [_I, _I, _P]),
    "txb_integrate_cells_host": (_I, [_I, _I, _I, _I, _I, _I, _I, c_int64] + [_P] * 8 + [_I, _I]),
    "txb_integrate_mesh": (_I, [_I, _I, _I, _I, _I, _I, c_int64, c_int64] + [_P] * 11 + [_I, _P]),
    "txb_tile_counts": (_I, [_I, c_int64, _P, _I, _P, _P]),
    "txb_tile_build": (_I, [_I, c_int64, _P, _I, _I, _I, _P, _P, _P]),
    "txb_integrate_mesh_tiled": (_I, [_I, _I, _I, _I, _I, _I, c_int64, c_int64, _P, _P, _P, _P, _I, _P, _I, _P,
                                      _I, _P, _P, _P, _P, _P, _P, _P]),
    "txb_debug_geometry_fast": (_I, [_I, c_int64, _P, _P, _P, _P, _P, _I, _P]),
    "txb_debug_geometry_fast32": (_I, [_I, c_int64, _P, _P, _P, _P, _P, _P]),
    "txb_gather_coefficients": (_I, [_I, c_int64, _I, _I, _P, _P, _P, _P]),
    "txb_scatter_add": (_I, [_I, c_int64, _I, _P, _P, _P, _P, _P]),
    "txb_scatter_add_slots": (_I, [_I, c_int64, _I, _P, _P, _P, _P, _P, _P]),
    "txb_scatter_order_scratch_bytes": (c_int64, [c_int64]),
    "txb_build_scatter_order": (_I, [c_int64, c_int64, _P, _P, _P, _P, _P, _P, _P]),
    "txb_incidence_scratch_bytes": (c_int64, [c_int64, _I, c_int64]),
    "txb_build_incidence": (_I, [c_int64, _I, c_int64, _P, _P, _P, _P, _P]),
    "txb_compute_geometry": (_I, [_I, c_int64, _P, _P, _P, _P, POINTER(c_int64), _P]),
    "txb_stream_probe": (_I, [_P, c_int64, _P, c_int64, _P]),
    "txb_debug_trace": (_I, [_P, c_int64]),
    "txb_halo_window_bytes": (c_int64, [c_int64, _I, _I]),
    "txb_halo_window_alloc": (_I, [c_int64, POINTER(c_void_p), _P]),
    "txb_halo_window_open": (_I, [_P, POINTER(c_void_p)]),
    "txb_halo_window_close": (_I, [_P]),
    "txb_halo_window_free": (_I, [_P]),
    "txb_halo_window_error": (_I, [_P, POINTER(c_int)]),
    "txb_halo_put": (_I, [_I, _I, _I, _I, c_int64, _P, _P, _P, _P, _P, _P, _P, _I, ctypes.c_uint64, _P]),
    "txb_halo_assemble": (_I, [_I, _I, _I, _I, c_int64, _P, _P, c_int64, _P, _P, c_int64, _P, _I,
                               ctypes.c_uint64, _P, _P]),
    "txb_jit_compile": (_I, [c_char_p, c_char_p, c_char_p, _I, _I, _I, _I, _I, _I, _I, POINTER(c_void_p)]),
    "txb_jit_source": (c_char_p, [_P]),
    "txb_jit_log": (c_char_p, [_P]),
    "txb_jit_cubin_bytes": (c_int64, [_P]),
    "txb_jit_cubin": (c_int64, [_P, _P, c_int64]),
    "txb_jit_integrate": (_I, [_P, c_int64] + [_P] * 8 + [_I, _I, _P]),
    "txb_jit_integrate_mesh": (_I, [_P, c_int64, c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P]),
    "txb_jit_integrate_mesh_tiled": (_I, [_P, c_int64, c_int64, _P, _P, _P, _P, _I, _P, _I, _P, _I, _P, _P, _P,
                                          _P, _P, _P, _P]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libtxb.so once; raise CudaLaneError if it is not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise CudaLaneError(
                f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            handle = ctypes.CDLL(str(LIB_PATH))
        except OSError as exc:  # pragma: no cover - environment dependent
            raise CudaLaneError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().txb_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int, what: str = "txb") -> None:
    """Map a C ABI return code onto the reference's exception classes."""
    if rc == TXB_OK:
        return
    msg = last_error() or what
    if rc == TXB_E_UNSUPPORTED:
        raise ValueError(f"cuda backend requested but unavailable for this configuration: {msg}")
    if rc == TXB_E_SHAPE:
        raise ShapeError(msg)
    if rc == TXB_E_CONFIG:
        raise ConfigurationError(msg)
    if rc == TXB_E_CAPACITY:
        nums = [int(x) for x in re.findall(r"needs (\d+) bytes, budget is (\d+)", msg)[0]] \
            if re.search(r"needs (\d+) bytes, budget is (\d+)", msg) else [0, 0]
        raise CapacityError(msg, required_bytes=nums[0], limit_bytes=nums[1])
    if rc == TXB_E_ORIENTATION:
        raise OrientationError(msg)
    if rc == TXB_E_ARG:
        raise ValueError(msg)
    if rc == TXB_E_COMPILE:
        raise CodegenError(msg)
    raise CudaLaneError(msg)
