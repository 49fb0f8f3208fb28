"""ctypes binding of libevsim_gpu.so (the C-ABI declared in include/evsim_gpu.h).

The library is built in-tree (paper_2209_04634_b200/build.py).  There is no
CPU fallback: if the shared object is missing or cannot be loaded, every
entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .abi import CConfig, CEvents, CWire

HERE = os.path.dirname(os.path.abspath(__file__))
# EVSIM_GPU_LIB=checked loads the bounds-checked build (build.py checked=True)
LIB_PATH = os.path.join(HERE, "libevsim_gpu_checked.so" if os.environ.get("EVSIM_GPU_LIB") == "checked"
                        else "libevsim_gpu.so")

_lock = threading.Lock()
_lib = None

_vp = ctypes.c_void_p
_i32, _i64 = ctypes.c_int32, ctypes.c_int64

_SIGS = {
    "evsim_gpu_last_error": (ctypes.c_char_p, []),
    "evsim_gpu_config_defaults": (None, [_i32, ctypes.POINTER(CConfig)]),
    "evsim_gpu_config_validate": (ctypes.c_int, [ctypes.POINTER(CConfig)]),
    "evsim_gpu_create": (ctypes.c_int, [ctypes.POINTER(CConfig), ctypes.c_int, ctypes.POINTER(_vp)]),
    "evsim_gpu_push_frame": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i64, _i32, ctypes.POINTER(CEvents)]),
    "evsim_gpu_push_frame_async": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i64, _i32]),
    "evsim_gpu_push_frames": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _i32, ctypes.POINTER(CEvents)]),
    "evsim_gpu_push_frames_async": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _i32]),
    "evsim_gpu_push_frames_batched": (
        ctypes.c_int, [_vp, _i32, _vp, _i32, _i32, _i32, _vp, _i32, ctypes.POINTER(CEvents)]),
    "evsim_gpu_push_frames_streamed": (
        ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _i32, _vp, _i64, ctypes.POINTER(CEvents)]),
    "evsim_gpu_push_frames_wire": (
        ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _i32, ctypes.POINTER(CWire), ctypes.POINTER(CEvents)]),
    "evsim_gpu_wire_unpack": (ctypes.c_int, [ctypes.POINTER(CWire), _i32, _vp, _i64, _i32]),
    "evsim_gpu_place_events": (ctypes.c_int, [_vp, _vp, _vp, _i32]),
    "evsim_gpu_ipc_handle": (ctypes.c_int, [_vp, _vp]),
    "evsim_gpu_ipc_open": (ctypes.c_int, [_i32, _vp, ctypes.POINTER(_vp)]),
    "evsim_gpu_ipc_close": (ctypes.c_int, [_i32, _vp]),
    "evsim_gpu_max_batch": (ctypes.c_int, [_vp, _i32, _i32]),
    "evsim_gpu_ingest_frames": (ctypes.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp]),
    "evsim_gpu_write_events_binary": (ctypes.c_int, [_vp, ctypes.c_char_p]),
    "evsim_gpu_write_events_text": (ctypes.c_int, [_vp, ctypes.c_char_p]),
    "evsim_gpu_events_per_pixel_second": (
        ctypes.c_int, [_vp, _i64, _i32, _i32, ctypes.c_double, ctypes.POINTER(ctypes.c_double),
                       ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]),
    "evsim_gpu_accumulate": (ctypes.c_int, [_vp, _i64, _i32, _i32, _i64, _i64, _vp]),
    "evsim_gpu_difference_frame": (ctypes.c_int, [_vp, _vp, _i32, _i32, _vp]),
    "evsim_gpu_log_lut": (None, [_vp]),
    "evsim_gpu_push_frame_with_flow": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i64, _vp, _vp, ctypes.POINTER(CEvents)]),
    "evsim_gpu_push_frame_with_tracks": (
        ctypes.c_int, [_vp, _vp, _i32, _i32, _i64, _vp, _i64, _vp, _vp, ctypes.POINTER(CEvents)]),
    "evsim_gpu_threshold_events": (
        ctypes.c_int, [_vp, _i32, _i32, ctypes.POINTER(CConfig), _i64, _vp, _i64, ctypes.POINTER(_i64)]),
    "evsim_gpu_set_row_band": (ctypes.c_int, [_vp, _i32, _i32]),
    "evsim_gpu_sync": (ctypes.c_int, [_vp, ctypes.POINTER(CEvents)]),
    "evsim_gpu_copy_events": (ctypes.c_int, [_vp, _vp, _i64, _i32]),
    "evsim_gpu_stream": (_vp, [_vp]),
    "evsim_gpu_reset": (ctypes.c_int, [_vp]),
    "evsim_gpu_destroy": (None, [_vp]),
    "evsim_gpu_kernel_launches": (_i64, [_vp]),
    "evsim_gpu_set_profiling": (ctypes.c_int, [_vp, _i32]),
    "evsim_gpu_stage_times": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_double), _i32, ctypes.POINTER(_i64)]),
    "evsim_gpu_dense_flow": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "evsim_gpu_sparse_flow": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _i64, _vp, _vp]),
    "evsim_gpu_interpolate_frames": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i64, _i64, _vp, _vp, _i32, _vp, _vp]),
    "evsim_gpu_dense_events_with_flow": (
        ctypes.c_int, [_vp, _vp, _i32, _i32, _i64, _i64, _vp, _vp, ctypes.POINTER(CConfig), _vp, _i64,
                       ctypes.POINTER(_i64)]),
    "evsim_gpu_sparse_events_with_flow": (
        ctypes.c_int, [_vp, _vp, _i32, _i32, _i64, _i64, _vp, _i64, _vp, _vp, ctypes.POINTER(CConfig), _vp, _i64,
                       ctypes.POINTER(_i64)]),
}

EXPORTED = tuple(_SIGS)


def load(build_if_missing: bool = True):
    """Load (and, in a source checkout, build) the CUDA library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH) and build_if_missing:
            from .build import build
            build(checked=LIB_PATH.endswith("_checked.so"))
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA library missing: {LIB_PATH} (run paper_2209_04634_b200/build.py)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class EvsimError(RuntimeError):
    """Non-zero status from the C-ABI.  ``code`` is the EVSIM_GPU_* status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(EvsimError, ValueError):
    """EVSIM_GPU_INVALID_ARGUMENT — the reference's std::invalid_argument."""


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().evsim_gpu_last_error().decode()
    if rc == 1:
        raise InvalidArgument(rc, msg)
    raise EvsimError(rc, msg)
