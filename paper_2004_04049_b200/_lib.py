"""ctypes loader for libholo.so (the C ABI declared in include/holo.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind this library.  There is no CPU fallback -- if the library is
missing or cannot be loaded, ``lib()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libholo.so")
_lock = threading.Lock()
_lib = None

HOLO_OK, HOLO_ERR_INVALID_ARG, HOLO_ERR_UNSUPPORTED, HOLO_ERR_WORKSPACE, HOLO_ERR_CUDA = range(5)
STATUS_NAMES = {0: "HOLO_OK", 1: "HOLO_ERR_INVALID_ARG", 2: "HOLO_ERR_UNSUPPORTED",
                3: "HOLO_ERR_WORKSPACE", 4: "HOLO_ERR_CUDA"}


class HoloRegion(C.Structure):
    _fields_ = [("row0", C.c_int32), ("row1", C.c_int32), ("col0", C.c_int32), ("col1", C.c_int32)]


class HoloError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_vp = C.c_void_p
_i32 = C.c_int32
_u64 = C.c_uint64
_sz = C.c_size_t

# name -> (restype, argtypes); the complete exported surface of include/holo.h
SIGNATURES = {
    "holo_last_error": (C.c_char_p, []),
    "holo_version": (C.c_char_p, []),
    "holo_lut_generate": (C.c_int, [_u64, _u64, _vp, _vp]),
    "holo_ospr_workspace_size": (_sz, [_i32, _i32, _i32]),
    "holo_ospr_chunk_pairs": (_i32, [_i32, _i32]),
    "holo_ospr_finalize_workspace_size": (_sz, []),
    "holo_gs_group_frames": (_i32, [_i32, _i32]),
    "holo_ospr_generate": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _u64, _u64, _i32, _i32, _vp, _vp, _vp,
                                     HoloRegion, _vp, _sz, _vp]),
    "holo_ospr_generate_prng": (C.c_int, [_vp, _i32, _i32, _i32, _u64, _u64, _i32, _i32, _vp, _vp, _vp,
                                          HoloRegion, _vp, _sz, _vp]),
    "holo_phase_table": (C.c_int, [_i32, _vp, _vp]),
    "holo_ospr_generate_prng_table": (C.c_int, [_vp, _i32, _i32, _i32, _u64, _vp, _i32, _u64, _i32, _i32, _vp, _vp,
                                                _vp, HoloRegion, _vp, _sz, _vp]),
    "holo_ospr_finalize": (C.c_int, [_vp, _vp, _i32, _i32, _i32, HoloRegion, _vp, _vp, _vp, _sz, _vp]),
    "holo_ospr_finalize_rows": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, HoloRegion, _vp, _vp, _vp, _sz, _vp]),
    "holo_ospr_mse_from_sums": (C.c_int, [_vp, _i32, HoloRegion, _vp, _vp]),
    "holo_debug_ospr_pairs": (C.c_int, [_vp, _i32, _i32, _vp, _u64, _i32, _u64, _u64, _i32, _i32, _vp, _vp]),
    "holo_gs_workspace_size": (_sz, [_i32, _i32, _i32]),
    "holo_gs_generate": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _u64, _u64, _i32, _vp, _vp, _vp, _vp, _vp,
                                   HoloRegion, _vp, _sz, _vp]),
    "holo_fft2": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _vp]),
    "holo_debug_randomise": (C.c_int, [_vp, _i32, _vp, _u64, _u64, _vp, _vp]),
    "holo_gs_step": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, HoloRegion, _vp, _sz,
                               _vp]),
    "holo_ospr_stream_create": (C.c_int, [_i32, _i32, _i32, _vp, _u64, _i32, _u64, _u64, _u64, _i32, HoloRegion,
                                          _vp, _vp, _sz, C.POINTER(_vp)]),
    "holo_ospr_stream_submit": (C.c_int, [_vp, _vp, C.POINTER(C.c_int64)]),
    "holo_ospr_stream_wait": (C.c_int, [_vp, C.c_int64]),
    "holo_ospr_stream_done": (_i32, [_vp, C.c_int64]),
    "holo_ospr_stream_drain": (C.c_int, [_vp]),
    "holo_ospr_stream_destroy": (None, [_vp]),
    "holo_ospr_stream_handles": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)]),
    "holo_launch_count": (_u64, []),
    "holo_profile_enable": (C.c_int, [_i32]),
    "holo_profile_read": (C.c_int, [C.c_char_p, C.POINTER(_u64), C.POINTER(C.c_double)]),
    "holo_kernel_names": (C.c_char_p, []),
}


def lib():
    """Load libholo.so (raising if it is absent: there is no fallback path)."""
    global _lib
    if _lib is not None:                 # fast path: no lock once loaded
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} not found: build it with `python -m paper_2004_04049_b200.build` "
                    "(libholo is the only implementation; there is no CPU fallback)")
            h = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def check(status: int) -> None:
    if status != HOLO_OK:
        raise HoloError(status, lib().holo_last_error().decode())
