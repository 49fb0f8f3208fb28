"""ctypes mirror of include/evsim_gpu.h (the C-ABI boundary).

Pure data definitions shared by the host wrapper, the tests and the oracle
wrapper: the config struct (evsim::SimulatorConfig + extension fields,
reference include/evsim/types.hpp:88-131), the 24-byte event record
(evsim::Event, types.hpp:54-61) as a numpy dtype, and the enums.
"""
from __future__ import annotations

import ctypes
import enum

import numpy as np


class Method(enum.IntEnum):
    """evsim::Method (reference include/evsim/types.hpp:82)."""

    difference_only = 0
    dense = 1
    sparse = 2
    difference_interp = 3


class FlowQuality(enum.IntEnum):
    """evsim::FlowQuality (types.hpp:83)."""

    low_quality = 0
    high_quality = 1


class EventsPerCrossing(enum.IntEnum):
    """evsim::EventsPerCrossing (types.hpp:86)."""

    single = 0
    magnitude = 1


class ContrastMode(enum.IntEnum):
    """Extension: linear (reference semantics) or log intensity (BASELINE configs)."""

    linear = 0
    log = 1


STATUS_OK = 0
STATUS_INVALID_ARGUMENT = 1
STATUS_RUNTIME = 2
STATUS_CUDA = 3


class CConfig(ctypes.Structure):
    """struct evsim_gpu_config."""

    _fields_ = [
        ("method", ctypes.c_int32),
        ("c_pos", ctypes.c_int32),
        ("c_neg", ctypes.c_int32),
        ("n_interp", ctypes.c_int32),
        ("flow_preset", ctypes.c_int32),
        ("selection_threshold", ctypes.c_int32),
        ("events_per_crossing", ctypes.c_int32),
        ("include_endpoints", ctypes.c_int32),
        ("contrast_mode", ctypes.c_int32),
        ("c_pos_log", ctypes.c_float),
        ("c_neg_log", ctypes.c_float),
        ("sel_log", ctypes.c_float),
        ("pyramid_levels", ctypes.c_int32),
        ("iterations_per_level", ctypes.c_int32),
        ("patch_radius", ctypes.c_int32),
    ]


class CEvents(ctypes.Structure):
    """struct evsim_gpu_events."""

    _fields_ = [
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("n_events", ctypes.c_int64),
        ("n_segments", ctypes.c_int32),
        ("seg_t", ctypes.POINTER(ctypes.c_int64)),
        ("seg_offset", ctypes.POINTER(ctypes.c_int64)),
        ("d_packed", ctypes.c_void_p),
    ]


class CWire(ctypes.Structure):
    """struct evsim_gpu_wire (the compact lossless event wire format)."""

    _fields_ = [
        ("planes", ctypes.c_void_p),
        ("planes_capacity", ctypes.c_int64),
        ("polarity", ctypes.c_void_p),
        ("polarity_capacity", ctypes.c_int64),
        ("link_t", ctypes.c_void_p),
        ("link_events", ctypes.c_void_p),
        ("link_bit", ctypes.c_void_p),
        ("link_capacity", ctypes.c_int64),
        ("n_links", ctypes.c_int64),
        ("words_per_row", ctypes.c_int32),
        ("row0", ctypes.c_int32),
        ("rows", ctypes.c_int32),
        ("width", ctypes.c_int32),
        ("words_per_link", ctypes.c_int64),
        ("n_events", ctypes.c_int64),
        ("polarity_words", ctypes.c_int64),
    ]


# evsim::Event / evsim_event: x@0 u16, y@2 u16, t@8 i64, p@16 i8, sizeof 24.
EVENT_DTYPE = np.dtype(
    {"names": ["x", "y", "t", "p"], "formats": ["<u2", "<u2", "<i8", "i1"],
     "offsets": [0, 2, 8, 16], "itemsize": 24}
)


def defaults(method: Method) -> dict:
    """SimulatorConfig::defaults (reference types.hpp:101-120)."""
    m = Method(method)
    d = dict(method=int(m), c_pos=2, c_neg=-2, n_interp=0, flow_preset=0, selection_threshold=0,
             events_per_crossing=0, include_endpoints=1, contrast_mode=0, c_pos_log=0.2,
             c_neg_log=-0.2, sel_log=0.0, pyramid_levels=0, iterations_per_level=0,
             patch_radius=0)
    if m == Method.dense:
        d.update(c_pos=2, c_neg=-2, n_interp=10)
    elif m == Method.sparse:
        d.update(c_pos=10, c_neg=-10, n_interp=10, selection_threshold=10)
    elif m == Method.difference_interp:
        d.update(c_pos=20, c_neg=-20, n_interp=10)
    return d


def make_config(method: Method = Method.difference_only, **overrides) -> CConfig:
    d = defaults(method)
    for k, v in overrides.items():
        if k not in d:
            raise TypeError(f"unknown config field {k!r}")
        d[k] = int(v) if not isinstance(v, float) else v
    c = CConfig()
    for k, v in d.items():
        setattr(c, k, v)
    return c


def config_dict(c: CConfig) -> dict:
    return {name: getattr(c, name) for name, _ in CConfig._fields_}


def unpack_events(packed: np.ndarray, seg_t: np.ndarray, seg_offset: np.ndarray) -> np.ndarray:
    """Expand packed device records (x:16 | y:15 | neg:1) to evsim::Event records."""
    packed = np.asarray(packed, dtype=np.uint32)
    out = np.zeros(packed.shape[0], dtype=EVENT_DTYPE)
    out["x"] = packed & 0xFFFF
    out["y"] = (packed >> 16) & 0x7FFF
    out["p"] = np.where(packed >> 31, -1, 1)
    counts = np.diff(np.asarray(seg_offset, dtype=np.int64))
    out["t"] = np.repeat(np.asarray(seg_t, dtype=np.int64), counts)
    return out
