"""Host-side mirror of the reference `evsim` API over the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/evsim/{types,flow,simulate}.hpp), so code and
tests written against the reference read the same here:

* ``SimulatorConfig`` / ``SimulatorConfig.defaults``      types.hpp:88-131
* ``Frame``, ``EventStream``, ``FlowField``, ``SparseFlow`` types.hpp:14-80, flow.hpp:9-41
* ``FlowPreset`` / ``flow_preset``                          flow.hpp:45-59
* ``estimate_dense_flow`` / ``estimate_sparse_flow``        flow.hpp:64-70
* ``DenseFlowEstimator`` / ``SparseFlowEstimator`` plug-ins flow.hpp:74-110
* ``interpolate_frames``, ``dense_events_with_flow``,
  ``simulate_dense``, ``simulate_sparse``                   simulate.hpp:25-46
* ``Simulator`` (push_frame / reset / config)               simulate.hpp:60-94

Every compute call goes through libevsim_gpu.so (sm_100a kernels); there is
no CPU path.  Invalid arguments raise ``InvalidArgument`` (a ValueError)
carrying the reference's exact std::invalid_argument message.
"""
from __future__ import annotations

import ctypes
import dataclasses
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .abi import (EVENT_DTYPE, CConfig, CEvents, CWire, ContrastMode, EventsPerCrossing, FlowQuality, Method,
                  unpack_events)
from ._lib import EvsimError, InvalidArgument

_vp = ctypes.c_void_p


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


# --------------------------------------------------------------------------- types

@dataclasses.dataclass
class Frame:
    """evsim::Frame (types.hpp:14-34): u8 row-major pixels + timestamp (us)."""

    width: int
    height: int
    timestamp: int
    pixels: np.ndarray

    @classmethod
    def make(cls, width: int, height: int, timestamp: int = 0, fill: int = 0) -> "Frame":
        if width <= 0 or height <= 0:
            raise InvalidArgument(1, "Frame: width and height must be positive")
        return cls(width, height, timestamp, np.full((height, width), fill, np.uint8))

    @classmethod
    def from_array(cls, pixels: np.ndarray, timestamp: int) -> "Frame":
        pixels = np.ascontiguousarray(pixels, dtype=np.uint8)
        return cls(pixels.shape[1], pixels.shape[0], int(timestamp), pixels)


@dataclasses.dataclass
class EventStream:
    """evsim::EventStream (types.hpp:72-80); events use evsim::Event's layout."""

    width: int
    height: int
    events: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, EVENT_DTYPE))

    def append(self, other: "EventStream") -> None:
        self.events = np.concatenate([self.events, other.events])

    def __len__(self) -> int:
        return len(self.events)


@dataclasses.dataclass
class FlowPreset:
    """evsim::FlowPreset (flow.hpp:45-55)."""

    pyramid_levels: int = 3
    iterations_per_level: int = 2
    patch_radius: int = 4

    def validate(self) -> None:
        if self.pyramid_levels < 1 or self.iterations_per_level < 1 or self.patch_radius < 1:
            raise InvalidArgument(1, "FlowPreset: all fields must be >= 1")


def flow_preset(q: FlowQuality) -> FlowPreset:
    """flow.hpp:57-59."""
    return FlowPreset(3, 2, 4) if FlowQuality(q) == FlowQuality.low_quality else FlowPreset(5, 16, 6)


@dataclasses.dataclass
class FlowField:
    """evsim::FlowField (flow.hpp:9-23)."""

    width: int
    height: int
    du: np.ndarray
    dv: np.ndarray

    @classmethod
    def zeros(cls, width: int, height: int) -> "FlowField":
        return cls(width, height, np.zeros((height, width), np.float32), np.zeros((height, width), np.float32))


@dataclasses.dataclass
class SparseFlow:
    """evsim::SparseFlow (flow.hpp:37-41); points (M,2) int32 x,y."""

    points: np.ndarray
    displacements: np.ndarray  # (M, 2) float32 du, dv
    status: np.ndarray         # (M,) uint8, 1 tracked / 0 lost


@dataclasses.dataclass
class SimulatorConfig:
    """evsim::SimulatorConfig (types.hpp:88-131) + log-mode extension fields."""

    method: Method = Method.difference_only
    c_pos: int = 2
    c_neg: int = -2
    n_interp: int = 0
    flow_preset: FlowQuality = FlowQuality.low_quality
    selection_threshold: int = 0
    events_per_crossing: EventsPerCrossing = EventsPerCrossing.single
    include_endpoints: bool = True
    contrast_mode: ContrastMode = ContrastMode.linear
    c_pos_log: float = 0.2
    c_neg_log: float = -0.2
    sel_log: float = 0.0
    preset_override: Optional[FlowPreset] = None

    @classmethod
    def defaults(cls, m: Method) -> "SimulatorConfig":
        """SimulatorConfig::defaults (types.hpp:101-120)."""
        m = Method(m)
        c = cls(method=m)
        if m == Method.dense:
            c.c_pos, c.c_neg, c.n_interp = 2, -2, 10
        elif m == Method.sparse:
            c.c_pos, c.c_neg, c.n_interp, c.selection_threshold = 10, -10, 10, 10
        elif m == Method.difference_interp:
            c.c_pos, c.c_neg, c.n_interp = 20, -20, 10
        return c

    def effective_selection_threshold(self) -> int:
        return self.selection_threshold if self.selection_threshold > 0 else self.c_pos

    def to_c(self) -> CConfig:
        c = CConfig()
        c.method = int(self.method)
        c.c_pos = int(self.c_pos)
        c.c_neg = int(self.c_neg)
        c.n_interp = int(self.n_interp)
        c.flow_preset = int(self.flow_preset)
        c.selection_threshold = int(self.selection_threshold)
        c.events_per_crossing = int(self.events_per_crossing)
        c.include_endpoints = 1 if self.include_endpoints else 0
        c.contrast_mode = int(self.contrast_mode)
        c.c_pos_log = float(self.c_pos_log)
        c.c_neg_log = float(self.c_neg_log)
        c.sel_log = float(self.sel_log)
        if self.preset_override is not None:
            c.pyramid_levels = self.preset_override.pyramid_levels
            c.iterations_per_level = self.preset_override.iterations_per_level
            c.patch_radius = self.preset_override.patch_radius
        return c

    @classmethod
    def from_c(cls, c: CConfig) -> "SimulatorConfig":
        ov = None
        if c.pyramid_levels or c.iterations_per_level or c.patch_radius:
            ov = FlowPreset(c.pyramid_levels, c.iterations_per_level, c.patch_radius)
        return cls(method=Method(c.method), c_pos=c.c_pos, c_neg=c.c_neg, n_interp=c.n_interp,
                   flow_preset=FlowQuality(c.flow_preset), selection_threshold=c.selection_threshold,
                   events_per_crossing=EventsPerCrossing(c.events_per_crossing),
                   include_endpoints=bool(c.include_endpoints), contrast_mode=ContrastMode(c.contrast_mode),
                   c_pos_log=c.c_pos_log, c_neg_log=c.c_neg_log, sel_log=c.sel_log, preset_override=ov)

    def validate(self) -> None:
        """SimulatorConfig::validate (types.hpp:126-130), evaluated by the library."""
        c = self.to_c()
        _lib.check(_lib.load().evsim_gpu_config_validate(ctypes.byref(c)))

    def preset(self) -> FlowPreset:
        return self.preset_override if self.preset_override is not None else flow_preset(self.flow_preset)


# --------------------------------------------------------------------------- flow

def _check_pair(prev: Frame, curr: Frame, who: str, empty_check: bool = True) -> None:
    # check_pair, flow.cpp:249-256 / simulate.cpp:28-32
    if empty_check and (prev.width <= 0 or prev.height <= 0 or curr.width <= 0 or curr.height <= 0):
        raise InvalidArgument(1, f"{who}: empty frame")
    if prev.width != curr.width or prev.height != curr.height:
        raise InvalidArgument(1, f"{who}: incompatible input frames")


def estimate_dense_flow(prev: Frame, curr: Frame, preset: FlowPreset) -> FlowField:
    """estimate_dense_flow (flow.cpp:260-276) on the GPU."""
    preset.validate()
    _check_pair(prev, curr, "estimate_dense_flow")
    w, h = prev.width, prev.height
    du = np.zeros((h, w), np.float32)
    dv = np.zeros((h, w), np.float32)
    _lib.check(_lib.load().evsim_gpu_dense_flow(
        _ptr(prev.pixels), _ptr(curr.pixels), w, h, preset.pyramid_levels, preset.iterations_per_level,
        preset.patch_radius, _ptr(du), _ptr(dv)))
    return FlowField(w, h, du, dv)


def estimate_sparse_flow(prev: Frame, curr: Frame, points, preset: FlowPreset) -> SparseFlow:
    """estimate_sparse_flow (flow.cpp:278-381) on the GPU."""
    preset.validate()
    _check_pair(prev, curr, "estimate_sparse_flow")
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.int32).reshape(-1, 2))
    m = pts.shape[0]
    disp = np.zeros((m, 2), np.float32)
    st = np.zeros(m, np.uint8)
    _lib.check(_lib.load().evsim_gpu_sparse_flow(
        _ptr(prev.pixels), _ptr(curr.pixels), prev.width, prev.height, preset.pyramid_levels,
        preset.iterations_per_level, preset.patch_radius, _ptr(pts), m, _ptr(disp), _ptr(st)))
    return SparseFlow(pts, disp, st)


class DenseFlowEstimator:
    """Plug-in interface (flow.hpp:74-78)."""

    def estimate(self, prev: Frame, curr: Frame) -> FlowField:  # pragma: no cover - interface
        raise NotImplementedError


class SparseFlowEstimator:
    """Plug-in interface (flow.hpp:80-85)."""

    def estimate(self, prev: Frame, curr: Frame, points) -> SparseFlow:  # pragma: no cover
        raise NotImplementedError


class PyramidalPatchFlow(DenseFlowEstimator):
    """Default dense backend (flow.hpp:88-97), on the GPU."""

    def __init__(self, preset: FlowPreset):
        preset.validate()
        self.preset = preset

    def estimate(self, prev: Frame, curr: Frame) -> FlowField:
        return estimate_dense_flow(prev, curr, self.preset)


class PyramidalLucasKanade(SparseFlowEstimator):
    """Default sparse backend (flow.hpp:100-110), on the GPU."""

    def __init__(self, preset: FlowPreset):
        preset.validate()
        self.preset = preset

    def estimate(self, prev: Frame, curr: Frame, points) -> SparseFlow:
        return estimate_sparse_flow(prev, curr, points, self.preset)


# --------------------------------------------------------------------------- core.hpp

@dataclasses.dataclass
class DifferenceFrame:
    """Signed per-pixel delta (types.hpp:33-46); values int16 (h, w)."""
    width: int
    height: int
    t_start: int
    t_end: int
    values: np.ndarray


def difference_frame(prev: Frame, curr: Frame) -> DifferenceFrame:
    """difference_frame (core.cpp:5-19) on the GPU."""
    if prev.width != curr.width or prev.height != curr.height:
        raise InvalidArgument(1, f"difference_frame: incompatible input frames ({prev.width}x{prev.height} vs "
                                 f"{curr.width}x{curr.height})")
    out = np.zeros((prev.height, prev.width), np.int16)
    _lib.check(_lib.load().evsim_gpu_difference_frame(_ptr(prev.pixels), _ptr(curr.pixels), prev.width,
                                                      prev.height, _ptr(out)))
    return DifferenceFrame(prev.width, prev.height, prev.timestamp, curr.timestamp, out)


def threshold_events(diff: DifferenceFrame, config: SimulatorConfig, event_time: int) -> np.ndarray:
    """threshold_events (core.cpp:21-52) on the GPU: 24-byte event records, scan order."""
    c = config.to_c()
    v = np.ascontiguousarray(diff.values, np.int16)
    return _call_events(_lib.load().evsim_gpu_threshold_events, _ptr(v), diff.width, diff.height, ctypes.byref(c),
                        int(event_time))


# --------------------------------------------------------------------------- pipelines

def _events_from_c(events24: np.ndarray, n: int, w: int, h: int) -> EventStream:
    return EventStream(w, h, events24[:n].copy())


def interpolate_frames(prev: Frame, curr: Frame, flow: FlowField, n: int) -> list:
    """interpolate_frames (simulate.cpp:91-121) on the GPU."""
    _check_pair(prev, curr, "interpolate_frames", empty_check=False)
    if flow.width != prev.width or flow.height != prev.height:
        raise InvalidArgument(1, "interpolate_frames: flow dimensions do not match the frames")
    if n < 0:
        raise InvalidArgument(1, "interpolate_frames: n must be >= 0")
    w, h = prev.width, prev.height
    out = np.zeros((max(n, 1), h, w), np.uint8)
    ts = np.zeros(max(n, 1), np.int64)
    _lib.check(_lib.load().evsim_gpu_interpolate_frames(
        _ptr(prev.pixels), _ptr(curr.pixels), w, h, prev.timestamp, curr.timestamp,
        _ptr(np.ascontiguousarray(flow.du, np.float32)), _ptr(np.ascontiguousarray(flow.dv, np.float32)),
        n, _ptr(out), _ptr(ts)))
    return [Frame(w, h, int(ts[k]), out[k].copy()) for k in range(n)]


def _call_events(fn, *args) -> np.ndarray:
    n = ctypes.c_int64()
    _lib.check(fn(*args, None, 0, ctypes.byref(n)))
    buf = np.zeros(max(n.value, 1), EVENT_DTYPE)
    _lib.check(fn(*args, _ptr(buf), n.value, ctypes.byref(n)))
    return buf[: n.value]


def dense_events_with_flow(prev: Frame, curr: Frame, flow: FlowField, config: SimulatorConfig) -> EventStream:
    """dense_events_with_flow (simulate.cpp:123-128): caller-supplied flow, GPU chain."""
    config.validate()
    _check_pair(prev, curr, "interpolate_frames", empty_check=False)
    if flow.width != prev.width or flow.height != prev.height:
        raise InvalidArgument(1, "interpolate_frames: flow dimensions do not match the frames")
    c = config.to_c()
    ev = _call_events(_lib.load().evsim_gpu_dense_events_with_flow, _ptr(prev.pixels), _ptr(curr.pixels),
                      prev.width, prev.height, prev.timestamp, curr.timestamp,
                      _ptr(np.ascontiguousarray(flow.du, np.float32)),
                      _ptr(np.ascontiguousarray(flow.dv, np.float32)), ctypes.byref(c))
    return EventStream(prev.width, prev.height, ev)


def select_points(prev: Frame, curr: Frame, config: SimulatorConfig) -> np.ndarray:
    """Host restatement of simulate.cpp:149-159 (scan-order selection) — used
    only when a custom SparseFlowEstimator must receive the point list.  Log
    mode: |L[curr] - L[prev]| > sel_log in fp32 with the library's own table
    (evsim_gpu_log_lut), exactly as the device selection."""
    if config.contrast_mode == ContrastMode.log:
        lut = np.zeros(256, np.float32)
        _lib.load().evsim_gpu_log_lut(_ptr(lut))
        sel = np.float32(config.sel_log if config.sel_log > 0 else config.c_pos_log)
        d = np.abs(lut[curr.pixels] - lut[prev.pixels])  # float32 IEEE subtraction
        ys, xs = np.nonzero(d > sel)
    else:
        d = np.abs(curr.pixels.astype(np.int32) - prev.pixels.astype(np.int32))
        ys, xs = np.nonzero(d > config.effective_selection_threshold())
    return np.stack([xs, ys], axis=1).astype(np.int32)


def sparse_events_with_flow(prev: Frame, curr: Frame, flow: SparseFlow, config: SimulatorConfig) -> EventStream:
    """simulate_sparse after its estimator call (simulate.cpp:163-201), GPU splat + chain."""
    config.validate()
    c = config.to_c()
    pts = np.ascontiguousarray(np.asarray(flow.points, np.int32).reshape(-1, 2))
    ev = _call_events(_lib.load().evsim_gpu_sparse_events_with_flow, _ptr(prev.pixels), _ptr(curr.pixels),
                      prev.width, prev.height, prev.timestamp, curr.timestamp, _ptr(pts), pts.shape[0],
                      _ptr(np.ascontiguousarray(flow.displacements, np.float32)),
                      _ptr(np.ascontiguousarray(flow.status, np.uint8)), ctypes.byref(c))
    return EventStream(prev.width, prev.height, ev)


def simulate_dense(prev: Frame, curr: Frame, config: SimulatorConfig,
                   estimator: Optional[DenseFlowEstimator] = None) -> EventStream:
    """simulate_dense (simulate.cpp:130-143)."""
    config.validate()
    _check_pair(prev, curr, "simulate_dense", empty_check=False)
    if estimator is None or (isinstance(estimator, PyramidalPatchFlow) and estimator.preset == config.preset()):
        sim = Simulator(config)
        sim.push_frame(prev)
        return sim.push_frame(curr)
    if config.n_interp == 0:
        return dense_events_with_flow(prev, curr, FlowField.zeros(prev.width, prev.height), config)
    return dense_events_with_flow(prev, curr, estimator.estimate(prev, curr), config)


def simulate_sparse(prev: Frame, curr: Frame, config: SimulatorConfig,
                    estimator: Optional[SparseFlowEstimator] = None) -> EventStream:
    """simulate_sparse (simulate.cpp:145-206)."""
    config.validate()
    _check_pair(prev, curr, "simulate_sparse", empty_check=False)
    if estimator is None or (isinstance(estimator, PyramidalLucasKanade) and estimator.preset == config.preset()):
        sim = Simulator(config)
        sim.push_frame(prev)
        return sim.push_frame(curr)
    pts = select_points(prev, curr, config)
    if len(pts) == 0 or config.n_interp == 0:
        return sparse_events_with_flow(prev, curr, SparseFlow(pts, np.zeros((0, 2), np.float32),
                                                               np.zeros(0, np.uint8)), config)
    return sparse_events_with_flow(prev, curr, estimator.estimate(prev, curr, pts), config)


def simulate_difference(f0: Frame, f1: Frame, f2: Frame, config: SimulatorConfig,
                        estimator: Optional[SparseFlowEstimator] = None) -> EventStream:
    """simulate_difference (simulate.cpp:287-301): the difference_interp events
    of (f1, f2] from the difference frames f1 - f0 and f2 - f1."""
    config.validate()
    _check_pair(f0, f1, "simulate_difference", empty_check=False)
    _check_pair(f1, f2, "simulate_difference", empty_check=False)
    if not (f0.timestamp < f1.timestamp < f2.timestamp):
        raise InvalidArgument(1, "simulate_difference: timestamps must be strictly increasing")
    if estimator is not None and not (isinstance(estimator, PyramidalLucasKanade)
                                      and estimator.preset == config.preset()):
        raise InvalidArgument(1, "simulate_difference: custom sparse estimators are not supported on the GPU path")
    sim = Simulator(dataclasses.replace(config, method=Method.difference_interp))
    sim.push_frame(f0)
    sim.push_frame(f1)
    return sim.push_frame(f2)


# --------------------------------------------------------------------------- Simulator

class Simulator:
    """evsim::Simulator (simulate.hpp:60-94) backed by one GPU handle.

    ``Simulator(config)`` runs the whole push on the device.  Passing custom
    ``dense_flow`` / ``sparse_flow`` estimators (the reference's plug-in seam,
    simulate.hpp:68-77) routes the flow through them; the stream's state and
    everything else stay on the device (both contrast modes).
    """

    def __init__(self, config: SimulatorConfig, dense_flow: Optional[DenseFlowEstimator] = None,
                 sparse_flow: Optional[SparseFlowEstimator] = None, device: int = 0, _null_check: bool = False):
        config.validate()
        if _null_check and (dense_flow is None or sparse_flow is None):
            raise InvalidArgument(1, "Simulator: flow estimators must not be null")
        self._config = dataclasses.replace(config)
        self._custom = (dense_flow is not None and not isinstance(dense_flow, PyramidalPatchFlow)) or \
                       (sparse_flow is not None and not isinstance(sparse_flow, PyramidalLucasKanade))
        if self._custom and Method(config.method) == Method.difference_interp:
            raise InvalidArgument(1, "Simulator: custom flow estimators are not supported for difference_interp")
        self._dense, self._sparse = dense_flow, sparse_flow
        self._lib = _lib.load()
        self._h = _vp()
        self._prev: Optional[Frame] = None
        c = config.to_c()
        _lib.check(self._lib.evsim_gpu_create(ctypes.byref(c), device, ctypes.byref(self._h)))

    @property
    def config(self) -> SimulatorConfig:
        return self._config

    def push_frame(self, frame: Frame) -> EventStream:
        """Simulator::push_frame (simulate.cpp:306-347)."""
        pixels = np.ascontiguousarray(frame.pixels, dtype=np.uint8)
        if frame.width <= 0 or frame.height <= 0 or pixels.size != frame.width * frame.height:
            raise InvalidArgument(1, "push_frame: malformed frame")
        if self._custom:
            return self._push_custom(frame, pixels)
        ev = CEvents()
        _lib.check(self._lib.evsim_gpu_push_frame(self._h, _ptr(pixels), frame.width, frame.height,
                                                  int(frame.timestamp), 0, ctypes.byref(ev)))
        return self._collect(ev)

    def _collect(self, ev: CEvents) -> EventStream:
        n = ev.n_events
        out = EventStream(ev.width, ev.height)
        if n == 0:
            return out
        packed = np.zeros(n, np.uint32)
        _lib.check(self._lib.evsim_gpu_copy_events(self._h, _ptr(packed), n, 0))
        S = ev.n_segments
        seg_t = np.ctypeslib.as_array(ev.seg_t, shape=(S,)).copy()
        seg_off = np.ctypeslib.as_array(ev.seg_offset, shape=(S + 1,)).copy()
        out.events = unpack_events(packed, seg_t, seg_off)
        return out

    def write_events_binary(self, path: str) -> None:
        """write_events_binary (io.cpp:148-170) of the last push's events,
        records formatted on the device."""
        _lib.check(self._lib.evsim_gpu_write_events_binary(self._h, str(path).encode()))

    def write_events_text(self, path: str) -> None:
        """write_events_text (io.cpp:105-126) of the last push's events."""
        _lib.check(self._lib.evsim_gpu_write_events_text(self._h, str(path).encode()))

    def set_row_band(self, y0: int, y1: int) -> None:
        """Emit only the events of rows [y0, y1) (evsim_gpu_set_row_band);
        (0, 0) = whole frame.  Stream start only; dense / difference_only."""
        _lib.check(self._lib.evsim_gpu_set_row_band(self._h, int(y0), int(y1)))

    def max_batch(self, width: int, height: int) -> int:
        """Largest push_frames batch for this config at width x height."""
        return int(self._lib.evsim_gpu_max_batch(self._h, width, height))

    def push_frames(self, frames: np.ndarray, timestamps) -> EventStream:
        """Batched push: identical to push_frame over each frame, events
        concatenated.  frames: (F, H, W) uint8; timestamps: F ints.  Batches
        larger than max_batch are split."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        ts = np.ascontiguousarray(np.asarray(timestamps, dtype=np.int64))
        F, h, w = frames.shape
        if self._custom:
            return concatenate([self.push_frame(Frame(w, h, int(ts[k]), frames[k])) for k in range(F)])
        parts = []
        step = self.max_batch(w, h)
        for a in range(0, F, step):
            b = min(F, a + step)
            ev = CEvents()
            _lib.check(self._lib.evsim_gpu_push_frames(self._h, _ptr(frames[a:b]), b - a, w, h, _ptr(ts[a:b]), 0,
                                                       ctypes.byref(ev)))
            parts.append(self._collect(ev))
        out = concatenate(parts)
        out.width, out.height = w, h
        return out

    def push_frames_streamed(self, frames: np.ndarray, timestamps, chunk: int = 0,
                             out: Optional[np.ndarray] = None) -> tuple:
        """Host frames in, host events out, upload / compute / download
        overlapped (evsim_gpu_push_frames_streamed).  Returns (packed u32
        records, seg_t, seg_offset); the same events push_frames returns, in
        packed form (abi.unpack_events expands them).  `out` may be a
        pre-allocated (ideally pinned) u32 buffer."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        ts = np.ascontiguousarray(np.asarray(timestamps, dtype=np.int64))
        F, h, w = frames.shape
        if out is None:
            links = max(1, self.config.n_interp + 1)
            out = np.empty(F * h * w * links, dtype=np.uint32)
        ev = CEvents()
        _lib.check(self._lib.evsim_gpu_push_frames_streamed(self._h, _ptr(frames), F, w, h, _ptr(ts), int(chunk),
                                                            _ptr(out), out.size, ctypes.byref(ev)))
        n = int(ev.n_events)
        S = int(ev.n_segments)
        seg_t = np.ctypeslib.as_array(ev.seg_t, shape=(S,)).copy() if S else np.zeros(0, np.int64)
        seg_off = np.ctypeslib.as_array(ev.seg_offset, shape=(S + 1,)).copy() if S else np.zeros(1, np.int64)
        return out[:n], seg_t, seg_off

    def push_frames_streamed_ptr(self, pixels_ptr: int, n_frames: int, width: int, height: int, timestamps,
                                 events_ptr: int, capacity: int, chunk: int = 0) -> CEvents:
        """Raw-pointer form of push_frames_streamed (pinned host buffers)."""
        ts = np.ascontiguousarray(np.asarray(timestamps, dtype=np.int64))
        ev = CEvents()
        _lib.check(self._lib.evsim_gpu_push_frames_streamed(self._h, _vp(pixels_ptr), n_frames, width, height,
                                                            _ptr(ts), int(chunk), _vp(events_ptr), int(capacity),
                                                            ctypes.byref(ev)))
        return ev

    def push_frames_wire(self, frames: np.ndarray, timestamps, chunk: int = 0,
                         wire: Optional["WireBuffer"] = None) -> "WireBuffer":
        """Host frames in, the events in the compact wire format out
        (evsim_gpu_push_frames_wire; include/evsim_gpu.h): one plane bit per
        pixel-link + one polarity bit per event.  WireBuffer.unpack() gives
        the packed / 24-byte stream push_frames would return."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        F, h, w = frames.shape
        if wire is None:
            wire = WireBuffer.for_call(self, F, w, h)
        return wire.run(self, frames.ctypes.data, F, w, h, timestamps, chunk)

    def push_frames_device(self, pixels_ptr: int, n_frames: int, width: int, height: int, timestamps,
                           on_device: bool = True, sync: bool = True) -> Optional[CEvents]:
        """Device-resident batched push (no event download)."""
        ts = np.ascontiguousarray(np.asarray(timestamps, dtype=np.int64))
        if sync:
            ev = CEvents()
            _lib.check(self._lib.evsim_gpu_push_frames(self._h, _vp(pixels_ptr), n_frames, width, height, _ptr(ts),
                                                       1 if on_device else 0, ctypes.byref(ev)))
            return ev
        _lib.check(self._lib.evsim_gpu_push_frames_async(self._h, _vp(pixels_ptr), n_frames, width, height,
                                                         _ptr(ts), 1 if on_device else 0))
        return None

    def push_frame_packed(self, pixels_ptr: int, width: int, height: int, timestamp: int,
                          on_device: bool = True) -> CEvents:
        """Device-resident push (no event download): returns the C result struct."""
        ev = CEvents()
        _lib.check(self._lib.evsim_gpu_push_frame(self._h, _vp(pixels_ptr), width, height, int(timestamp),
                                                  1 if on_device else 0, ctypes.byref(ev)))
        return ev

    def push_frame_async(self, pixels_ptr: int, width: int, height: int, timestamp: int,
                         on_device: bool = True) -> None:
        _lib.check(self._lib.evsim_gpu_push_frame_async(self._h, _vp(pixels_ptr), width, height, int(timestamp),
                                                        1 if on_device else 0))

    def sync(self) -> CEvents:
        ev = CEvents()
        _lib.check(self._lib.evsim_gpu_sync(self._h, ctypes.byref(ev)))
        return ev

    def copy_packed(self, dst_ptr: int, capacity: int) -> None:
        _lib.check(self._lib.evsim_gpu_copy_events(self._h, _vp(dst_ptr), capacity, 0))

    def place_events(self, dst_ptr: int, dst_offsets) -> None:
        """evsim_gpu_place_events: segment s of the last push to
        dst + dst_offsets[s] records (device memory of this or a peer GPU,
        e.g. rank 0's merged buffer opened with parallel.open_shared)."""
        off = np.ascontiguousarray(np.asarray(dst_offsets, dtype=np.int64))
        _lib.check(self._lib.evsim_gpu_place_events(self._h, _vp(dst_ptr), _ptr(off), int(off.size)))

    def copy_events(self, dst_ptr: int, capacity: int, fmt: int) -> None:
        """evsim_gpu_copy_events: the last push's events to host memory in
        format 0 (packed), 1 (evsim_event, 24 B) or 2 (.evs, 13 B)."""
        _lib.check(self._lib.evsim_gpu_copy_events(self._h, _vp(dst_ptr), capacity, int(fmt)))

    @property
    def stream(self) -> int:
        return self._lib.evsim_gpu_stream(self._h) or 0

    STAGES = ("upload", "pyramid", "flow", "chain", "scan", "emit")

    def set_profiling(self, enable: bool) -> None:
        _lib.check(self._lib.evsim_gpu_set_profiling(self._h, 1 if enable else 0))

    def stage_times(self) -> tuple[dict, int]:
        """Accumulated device ms per pipeline stage and the number of timed pushes."""
        ms = (ctypes.c_double * len(self.STAGES))()
        n = ctypes.c_int64()
        _lib.check(self._lib.evsim_gpu_stage_times(self._h, ms, len(self.STAGES), ctypes.byref(n)))
        return {k: ms[i] for i, k in enumerate(self.STAGES)}, n.value

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.evsim_gpu_kernel_launches(self._h))

    def _push_custom(self, frame: Frame, pixels: np.ndarray) -> EventStream:
        """push_frame with the flow from the caller's estimators: the flow on
        the host (the estimator), the stream's state — prev frame, log
        reference state — and everything else on the device
        (evsim_gpu_push_frame_with_flow / _with_tracks), so log mode works
        through the seam too."""
        prev = self._prev
        f = Frame(frame.width, frame.height, int(frame.timestamp), pixels)
        if prev is not None:
            if frame.width != prev.width or frame.height != prev.height:
                raise InvalidArgument(1, "push_frame: frame dimensions changed mid-stream")
            if frame.timestamp <= prev.timestamp:
                raise InvalidArgument(1, "push_frame: timestamps must be strictly increasing")
        cfg = self._config
        m, n = Method(cfg.method), cfg.n_interp
        ev = CEvents()
        w, h, t = frame.width, frame.height, int(frame.timestamp)
        if m == Method.sparse and n > 0:
            pts = np.zeros((0, 2), np.int32)
            disp = np.zeros((0, 2), np.float32)
            st = np.zeros(0, np.uint8)
            if prev is not None:
                pts = select_points(prev, f, cfg)
                if len(pts):
                    fl = (self._sparse or PyramidalLucasKanade(cfg.preset())).estimate(prev, f, pts)
                    disp = np.ascontiguousarray(fl.displacements, np.float32).reshape(-1, 2)
                    st = np.ascontiguousarray(fl.status, np.uint8)
            pts = np.ascontiguousarray(pts, np.int32)
            _lib.check(self._lib.evsim_gpu_push_frame_with_tracks(
                self._h, _ptr(pixels), w, h, t, _ptr(pts), len(pts), _ptr(disp), _ptr(st), ctypes.byref(ev)))
        else:
            du = dv = None
            if prev is not None and m == Method.dense and n > 0:
                fl = (self._dense or PyramidalPatchFlow(cfg.preset())).estimate(prev, f)
                du = np.ascontiguousarray(fl.du, np.float32)
                dv = np.ascontiguousarray(fl.dv, np.float32)
            _lib.check(self._lib.evsim_gpu_push_frame_with_flow(
                self._h, _ptr(pixels), w, h, t, None if du is None else _ptr(du), None if dv is None else _ptr(dv),
                ctypes.byref(ev)))
        self._prev = f
        return self._collect(ev)

    def reset(self) -> None:
        """Simulator::reset (simulate.hpp:83-86)."""
        self._prev = None
        _lib.check(self._lib.evsim_gpu_reset(self._h))

    def close(self) -> None:
        if self._h:
            self._lib.evsim_gpu_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class WireBuffer:
    """Host buffers of evsim_gpu_wire (pinned when torch is available, so the
    downloads overlap the compute) sized for one call of F frames."""

    def __init__(self, n_links: int, words_per_link: int, max_events: int, pinned: bool = True):
        def buf(n, dt):
            if pinned:
                try:
                    import torch
                    t = torch.empty(max(int(n), 1), dtype={np.uint32: torch.int32, np.int64: torch.int64}[dt])
                    t = t.pin_memory()
                    self._keep.append(t)
                    return t.numpy().view(dt)
                except Exception:
                    pass
            return np.zeros(max(int(n), 1), dt)
        self._keep = []
        self.planes = buf(n_links * words_per_link, np.uint32)
        self.polarity = buf(max_events // 32 + 64 + 2 * n_links, np.uint32)
        self.link_t = buf(n_links, np.int64)
        self.link_events = buf(n_links, np.int64)
        self.link_bit = buf(n_links, np.int64)
        self.c = CWire()

    @classmethod
    def for_call(cls, sim: "Simulator", F: int, w: int, h: int, rows: Optional[int] = None) -> "WireBuffer":
        links = max(1, sim.config.n_interp + 1) * F
        rows = h if rows is None else rows
        wpl = rows * ((w + 31) // 32)
        return cls(links, wpl, links * rows * w)

    def run(self, sim, pixels_ptr: int, F: int, w: int, h: int, timestamps, chunk: int = 0) -> "WireBuffer":
        ts = np.ascontiguousarray(np.asarray(timestamps, dtype=np.int64))
        c = self.c
        c.planes, c.planes_capacity = self.planes.ctypes.data, self.planes.size
        c.polarity, c.polarity_capacity = self.polarity.ctypes.data, self.polarity.size
        c.link_t, c.link_events, c.link_bit = (self.link_t.ctypes.data, self.link_events.ctypes.data,
                                               self.link_bit.ctypes.data)
        c.link_capacity = self.link_t.size
        ev = CEvents()
        _lib.check(sim._lib.evsim_gpu_push_frames_wire(sim._h, _vp(pixels_ptr), F, w, h, _ptr(ts), int(chunk),
                                                       ctypes.byref(c), ctypes.byref(ev)))
        return self

    @property
    def n_events(self) -> int:
        return int(self.c.n_events)

    @property
    def bytes(self) -> int:
        """Host bytes the call delivered (planes + polarity words + link tables)."""
        c = self.c
        return 4 * int(c.n_links) * int(c.words_per_link) + 4 * int(c.polarity_words) + 24 * int(c.n_links)

    def unpack(self, fmt: int = 0, threads: int = 0) -> np.ndarray:
        """The reference's event stream: packed u32 records (fmt 0) or
        evsim::Event records (fmt 1, EVENT_DTYPE)."""
        n = self.n_events
        out = np.zeros(max(n, 1), np.uint32 if fmt == 0 else EVENT_DTYPE)
        _lib.check(_lib.load().evsim_gpu_wire_unpack(ctypes.byref(self.c), fmt, _ptr(out), n, int(threads)))
        return out[:n]

    def segments(self) -> tuple:
        """(seg_t, seg_offset) of the unpacked stream: links with equal
        timestamps merged, empty segments dropped."""
        L = int(self.c.n_links)
        t = self.link_t[:L]
        e = self.link_events[:L]
        if L == 0:
            return np.zeros(0, np.int64), np.zeros(1, np.int64)
        starts = np.concatenate([[True], t[1:] != t[:-1]])
        seg_t = t[starts]
        cnt = np.add.reduceat(e, np.nonzero(starts)[0])
        keep = cnt > 0
        off = np.concatenate([[0], np.cumsum(cnt[keep])]).astype(np.int64)
        return seg_t[keep].astype(np.int64), off


def concatenate(streams: Sequence[EventStream]) -> EventStream:
    if not streams:
        return EventStream(0, 0)
    out = EventStream(streams[0].width, streams[0].height)
    out.events = np.concatenate([s.events for s in streams]) if streams else out.events
    return out


def push_frames_batched(sims: Sequence["Simulator"], frames: Sequence[np.ndarray], timestamps) -> list:
    """Several independent streams in one call (evsim_gpu_push_frames_batched):
    sims[i] gets frames[i] ((F, H, W) uint8, the same F, H, W for all) with
    timestamps[i].  The pushes run concurrently on the handles' CUDA streams;
    returns one EventStream per simulator.  All batches are validated first:
    an invalid one rejects the call and leaves every stream untouched."""
    n = len(sims)
    if len(frames) != n or len(timestamps) != n:
        raise InvalidArgument(1, "push_frames_batched: one frame batch and one timestamp list per simulator")
    if n == 0:
        return []
    if any(s._custom for s in sims):
        return [s.push_frames(f, t) for s, f, t in zip(sims, frames, timestamps)]
    fr = [np.ascontiguousarray(f, dtype=np.uint8) for f in frames]
    ts = [np.ascontiguousarray(np.asarray(t, dtype=np.int64)) for t in timestamps]
    F, h, w = fr[0].shape
    for f, t in zip(fr, ts):
        if f.shape != (F, h, w) or t.shape != (F,):
            raise InvalidArgument(1, "push_frames_batched: every stream needs the same batch shape")
    lib = sims[0]._lib
    hs = (ctypes.c_void_p * n)(*[s._h.value for s in sims])
    px = (ctypes.c_void_p * n)(*[f.ctypes.data for f in fr])
    tp = (ctypes.c_void_p * n)(*[t.ctypes.data for t in ts])
    outs = (CEvents * n)()
    _lib.check(lib.evsim_gpu_push_frames_batched(hs, n, px, F, w, h, tp, 0, outs))
    res = []
    for s, ev in zip(sims, outs):
        r = s._collect(ev)
        r.width, r.height = w, h
        res.append(r)
    return res


def push_frames_batched_device(sims: Sequence["Simulator"], pixel_ptrs: Sequence[int], n_frames: int, width: int,
                               height: int, timestamps, on_device: bool = True) -> list:
    """Raw-pointer form of push_frames_batched (frames already in device or
    pinned host memory): returns one CEvents per simulator (device-resident
    events, valid until that handle's next push)."""
    n = len(sims)
    ts = [np.ascontiguousarray(np.asarray(t, dtype=np.int64)) for t in timestamps]
    lib = sims[0]._lib
    hs = (ctypes.c_void_p * n)(*[s._h.value for s in sims])
    px = (ctypes.c_void_p * n)(*[int(p) for p in pixel_ptrs])
    tp = (ctypes.c_void_p * n)(*[t.ctypes.data for t in ts])
    outs = (CEvents * n)()
    _lib.check(lib.evsim_gpu_push_frames_batched(hs, n, px, n_frames, width, height, tp, 1 if on_device else 0,
                                                 outs))
    return list(outs)


# --------------------------------------------------------------------------- data formats

def ingest_frames(src: np.ndarray, target: Optional[tuple] = None) -> np.ndarray:
    """load_frames' pixel path (io.cpp:41-103) on the GPU: (n, h, w) gray or
    (n, h, w, 3) RGB u8 frames -> luma_bt601 -> resize_bilinear to
    target = (width, height) -> (n, th, tw) u8."""
    a = np.ascontiguousarray(src, dtype=np.uint8)
    if a.ndim == 2:
        a = a[None]
    channels = 3 if a.ndim == 4 else 1
    n, h, w = a.shape[:3]
    tw, th = (w, h) if target is None else (int(target[0]), int(target[1]))
    out = np.zeros((n, max(th, 0), max(tw, 0)), np.uint8)
    lib = _lib.load()
    _lib.check(lib.evsim_gpu_ingest_frames(_ptr(a), channels, w, h, n, tw, th, _ptr(out)))
    return out


@dataclasses.dataclass
class EventRateStats:
    """evsim::EventRateStats (metrics.hpp:9-14)."""
    mean_rate: float
    std_rate: float
    duration: float
    total_events: int


def _ev24(stream: EventStream) -> np.ndarray:
    ev = np.zeros(len(stream.events), EVENT_DTYPE)
    for k in ("x", "y", "t", "p"):
        ev[k] = stream.events[k]
    return ev


def events_per_pixel_second(stream: EventStream, duration: float) -> EventRateStats:
    """events_per_pixel_second (metrics.cpp:7-39): counts on the GPU."""
    ev = _ev24(stream)
    m, s, t = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint64()
    lib = _lib.load()
    _lib.check(lib.evsim_gpu_events_per_pixel_second(_ptr(ev), len(ev), stream.width, stream.height,
                                                     float(duration), ctypes.byref(m), ctypes.byref(s),
                                                     ctypes.byref(t)))
    return EventRateStats(m.value, s.value, float(duration), int(t.value))


def accumulate(stream: EventStream, t_start: int, t_end: int) -> np.ndarray:
    """accumulate (metrics.cpp:41-69): (height, width) PixelClass codes
    (0 none, 1 positive, 2 negative, 3 both) over [t_start, t_end)."""
    ev = _ev24(stream)
    out = np.zeros((max(stream.height, 0), max(stream.width, 0)), np.uint8)
    lib = _lib.load()
    _lib.check(lib.evsim_gpu_accumulate(_ptr(ev), len(ev), stream.width, stream.height, int(t_start), int(t_end),
                                        _ptr(out)))
    return out
