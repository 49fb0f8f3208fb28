"""TEST INFRASTRUCTURE ONLY — CPU oracles for the event-simulation hot path.

* ``Oracle``: ctypes wrapper of oracle/libevsim_oracle.so, the plain-C
  restatement of the reference (oracle/evsim_oracle.c).
* ``Reference``: ctypes wrapper of oracle/_ref/libevsim_ref.so, the unmodified
  reference sources compiled in place (oracle/Makefile, oracle/ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product library
(paper_2209_04634_b200) never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from paper_2209_04634_b200.abi import EVENT_DTYPE, CConfig, make_config  # noqa: F401

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libevsim_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libevsim_ref.so")
REF_SRC = "/root/reference/proj"

_P = ctypes.POINTER
_u8p = ctypes.c_void_p
_i32, _i64, _f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build(ref: bool | None = None) -> None:
    """Compile the C restatement (and, when /root/reference exists, the
    reference and the reference's own unit suites against the drop-in:
    oracle/Makefile `refsuite`, after the CUDA library is built)."""
    targets = ["all"]
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        targets.append("ref")
        gpu_so = os.path.join(os.path.dirname(HERE), "paper_2209_04634_b200", "libevsim_gpu.so")
        if os.path.exists(gpu_so):
            targets += ["refsuite", "plugin"]
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _events(ptr, n) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=EVENT_DTYPE)
    buf = (ctypes.c_char * (24 * n)).from_address(ctypes.cast(ptr, ctypes.c_void_p).value)
    return np.frombuffer(buf, dtype=EVENT_DTYPE).copy()


class _Lib:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            build(ref=self.prefix == "evsim_ref")
        self.lib = ctypes.CDLL(self.path)
        p = self.prefix
        L = self.lib
        getattr(L, f"{p}_last_error").restype = ctypes.c_char_p
        self._err = getattr(L, f"{p}_last_error")

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._err().decode())

    # ---- stateless stages -------------------------------------------------
    def dense_flow(self, prev, curr, levels=3, iters=2, radius=4):
        h, w = prev.shape
        du = np.zeros((h, w), np.float32)
        dv = np.zeros((h, w), np.float32)
        self._check(getattr(self.lib, f"{self.prefix}_dense_flow")(
            _ptr(np.ascontiguousarray(prev)), _ptr(np.ascontiguousarray(curr)), _i32(w), _i32(h),
            _i32(levels), _i32(iters), _i32(radius), _ptr(du), _ptr(dv)))
        return du, dv

    def sparse_flow(self, prev, curr, pts, levels=3, iters=2, radius=4):
        h, w = prev.shape
        pts = np.ascontiguousarray(pts, dtype=np.int32).reshape(-1, 2)
        m = pts.shape[0]
        disp = np.zeros((m, 2), np.float32)
        st = np.zeros(m, np.uint8)
        self._check(getattr(self.lib, f"{self.prefix}_sparse_flow")(
            _ptr(np.ascontiguousarray(prev)), _ptr(np.ascontiguousarray(curr)), _i32(w), _i32(h),
            _i32(levels), _i32(iters), _i32(radius), _ptr(pts), _i64(m), _ptr(disp), _ptr(st)))
        return disp, st

    def interpolate_frames(self, prev, curr, t0, t1, du, dv, n):
        h, w = prev.shape
        out = np.zeros((max(n, 0), h, w), np.uint8)
        ts = np.zeros(max(n, 0), np.int64)
        self._check(getattr(self.lib, f"{self.prefix}_interpolate_frames")(
            _ptr(np.ascontiguousarray(prev)), _ptr(np.ascontiguousarray(curr)), _i32(w), _i32(h),
            _i64(t0), _i64(t1), _ptr(np.ascontiguousarray(du, np.float32)),
            _ptr(np.ascontiguousarray(dv, np.float32)), _i32(n), _ptr(out), _ptr(ts)))
        return out, ts


class Simulator:
    """Streaming simulator over either library (mirrors evsim::Simulator)."""

    def __init__(self, lib: _Lib, cfg: CConfig):
        self._lib = lib
        self._cfg = cfg
        h = ctypes.c_void_p()
        lib._check(getattr(lib.lib, f"{lib.prefix}_create")(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h

    def push_frame(self, pixels: np.ndarray, t: int) -> np.ndarray:
        pixels = np.ascontiguousarray(pixels, dtype=np.uint8)
        h, w = pixels.shape
        ev = ctypes.c_void_p()
        n = ctypes.c_int64()
        self._lib._check(getattr(self._lib.lib, f"{self._lib.prefix}_push_frame")(
            self._h, _ptr(pixels), _i32(w), _i32(h), _i64(t), ctypes.byref(ev), ctypes.byref(n)))
        return _events(ev, n.value)

    def reset(self):
        getattr(self._lib.lib, f"{self._lib.prefix}_reset")(self._h)

    def close(self):
        if self._h:
            getattr(self._lib.lib, f"{self._lib.prefix}_destroy")(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Oracle(_Lib):
    prefix = "evsim_oracle"
    path = ORACLE_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        L.evsim_oracle_ref_state.restype = ctypes.c_void_p

    def simulator(self, cfg: CConfig) -> Simulator:
        return Simulator(self, cfg)

    def log_lut(self) -> np.ndarray:
        lut = np.zeros(256, np.float32)
        self.lib.evsim_oracle_log_lut(_ptr(lut))
        return lut

    def dense_events_with_flow(self, prev, curr, t0, t1, du, dv, cfg: CConfig) -> np.ndarray:
        h, w = prev.shape
        ev = ctypes.c_void_p()
        n = ctypes.c_int64()
        self._check(self.lib.evsim_oracle_dense_events_with_flow(
            _ptr(np.ascontiguousarray(prev)), _ptr(np.ascontiguousarray(curr)), _i32(w), _i32(h),
            _i64(t0), _i64(t1), _ptr(np.ascontiguousarray(du, np.float32)),
            _ptr(np.ascontiguousarray(dv, np.float32)), ctypes.byref(cfg), ctypes.byref(ev),
            ctypes.byref(n)))
        out = _events(ev, n.value)
        self.lib.evsim_oracle_free(ev)
        return out

    def sparse_events_with_flow(self, prev, curr, t0, t1, pts, disp, status, cfg) -> np.ndarray:
        h, w = prev.shape
        pts = np.ascontiguousarray(pts, np.int32).reshape(-1, 2)
        ev = ctypes.c_void_p()
        n = ctypes.c_int64()
        self._check(self.lib.evsim_oracle_sparse_events_with_flow(
            _ptr(np.ascontiguousarray(prev)), _ptr(np.ascontiguousarray(curr)), _i32(w), _i32(h),
            _i64(t0), _i64(t1), _ptr(pts), _i64(pts.shape[0]),
            _ptr(np.ascontiguousarray(disp, np.float32)), _ptr(np.ascontiguousarray(status, np.uint8)),
            ctypes.byref(cfg), ctypes.byref(ev), ctypes.byref(n)))
        out = _events(ev, n.value)
        self.lib.evsim_oracle_free(ev)
        return out


class Reference(_Lib):
    prefix = "evsim_ref"
    path = REF_SO

    def run_sequence(self, cfg: CConfig, frames: np.ndarray, ts, threads: int):
        """Whole sequence on `threads` host threads with output identical to one
        streaming reference Simulator (ref_shim.cpp evsim_ref_run_sequence).
        Returns per-frame (counts int64[n], hashes uint64[n]) — the checksum of
        paper_2209_04634_b200/seqhash.py."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        n, h, w = frames.shape
        ts = np.ascontiguousarray(np.asarray(ts, dtype=np.int64))
        counts = np.zeros(n, np.int64)
        hashes = np.zeros(n, np.uint64)
        self._check(self.lib.evsim_ref_run_sequence(
            ctypes.byref(cfg), _ptr(frames), _i32(n), _i32(w), _i32(h), _ptr(ts), _i32(threads), _ptr(counts),
            _ptr(hashes)))
        return counts, hashes

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)

    def simulator(self, cfg: CConfig) -> Simulator:
        return Simulator(self, cfg)

    def dense_events_with_flow(self, prev, curr, t0, t1, du, dv, cfg: CConfig) -> np.ndarray:
        h, w = prev.shape
        ev = ctypes.c_void_p()
        n = ctypes.c_int64()
        self._check(self.lib.evsim_ref_dense_events_with_flow(
            _ptr(np.ascontiguousarray(prev)), _ptr(np.ascontiguousarray(curr)), _i32(w), _i32(h),
            _i64(t0), _i64(t1), _ptr(np.ascontiguousarray(du, np.float32)),
            _ptr(np.ascontiguousarray(dv, np.float32)), ctypes.byref(cfg), ctypes.byref(ev),
            ctypes.byref(n)))
        out = _events(ev, n.value)
        self.lib.evsim_ref_free(ev)
        return out

    def sparse_events_with_flow(self, prev, curr, t0, t1, disp, status, cfg) -> np.ndarray:
        h, w = prev.shape
        ev = ctypes.c_void_p()
        n = ctypes.c_int64()
        disp = np.ascontiguousarray(disp, np.float32).reshape(-1, 2)
        self._check(self.lib.evsim_ref_sparse_events_with_flow(
            _ptr(np.ascontiguousarray(prev)), _ptr(np.ascontiguousarray(curr)), _i32(w), _i32(h),
            _i64(t0), _i64(t1), _ptr(disp), _ptr(np.ascontiguousarray(status, np.uint8)),
            _i64(disp.shape[0]), ctypes.byref(cfg), ctypes.byref(ev), ctypes.byref(n)))
        out = _events(ev, n.value)
        self.lib.evsim_ref_free(ev)
        return out

    # ---- reference scenes (src/scenes.cpp) ----------------------------------
    def textured_frame(self, w, h, seed, lo=0, hi=255):
        out = np.zeros((h, w), np.uint8)
        self._check(self.lib.evsim_ref_textured_frame(_i32(w), _i32(h), ctypes.c_uint32(seed),
                                                      ctypes.c_uint8(lo), ctypes.c_uint8(hi), _ptr(out)))
        return out

    def panning_texture(self, w, h, n, dx, dy, fps=20.0, seed=1234):
        out = np.zeros((n, h, w), np.uint8)
        ts = np.zeros(n, np.int64)
        self._check(self.lib.evsim_ref_panning_texture(_i32(w), _i32(h), _i32(n), _i32(dx), _i32(dy),
                                                       ctypes.c_double(fps), ctypes.c_uint32(seed),
                                                       _ptr(out), _ptr(ts)))
        return out, ts

    def moving_disk(self, w, h, n, radius, step, fps, bg, fg, seed=0):
        out = np.zeros((n, h, w), np.uint8)
        ts = np.zeros(n, np.int64)
        self._check(self.lib.evsim_ref_moving_disk(_i32(w), _i32(h), _i32(n), ctypes.c_double(radius),
                                                   ctypes.c_double(step), ctypes.c_double(fps),
                                                   ctypes.c_uint8(bg), ctypes.c_uint8(fg),
                                                   ctypes.c_uint32(seed), _ptr(out), _ptr(ts)))
        return out, ts

    def translating_square(self, w, h, n, size, x0, y0, dx, dy, fps=30.0):
        out = np.zeros((n, h, w), np.uint8)
        ts = np.zeros(n, np.int64)
        self._check(self.lib.evsim_ref_translating_square(_i32(w), _i32(h), _i32(n), _i32(size),
                                                          _i32(x0), _i32(y0), _i32(dx), _i32(dy),
                                                          ctypes.c_double(fps), _ptr(out), _ptr(ts)))
        return out, ts

    # ---- frame ingestion, event files, metrics (src/io.cpp, src/metrics.cpp) --
    def luma(self, rgb: np.ndarray) -> np.ndarray:
        rgb = np.ascontiguousarray(rgb, np.uint8).reshape(-1, 3)
        f = self.lib.evsim_ref_luma_bt601
        f.restype = ctypes.c_uint8
        return np.array([f(ctypes.c_uint8(r), ctypes.c_uint8(g), ctypes.c_uint8(b)) for r, g, b in rgb], np.uint8)

    def resize_bilinear(self, frame: np.ndarray, tw: int, th: int) -> np.ndarray:
        h, w = frame.shape
        out = np.zeros((th, tw), np.uint8)
        self._check(self.lib.evsim_ref_resize_bilinear(_ptr(np.ascontiguousarray(frame, np.uint8)), _i32(w),
                                                       _i32(h), _i32(tw), _i32(th), _ptr(out)))
        return out

    @staticmethod
    def _ev24(events: np.ndarray) -> np.ndarray:
        from paper_2209_04634_b200.abi import EVENT_DTYPE
        out = np.zeros(len(events), EVENT_DTYPE)
        for k in ("x", "y", "t", "p"):
            out[k] = events[k]
        return out

    def write_events_binary(self, events: np.ndarray, w: int, h: int, path: str) -> None:
        ev = self._ev24(events)
        self._check(self.lib.evsim_ref_write_events_binary(_ptr(ev), _i64(len(ev)), _i32(w), _i32(h),
                                                           path.encode()))

    def write_events_text(self, events: np.ndarray, w: int, h: int, path: str) -> None:
        ev = self._ev24(events)
        self._check(self.lib.evsim_ref_write_events_text(_ptr(ev), _i64(len(ev)), _i32(w), _i32(h), path.encode()))

    def events_per_pixel_second(self, events: np.ndarray, w: int, h: int, duration: float):
        ev = self._ev24(events)
        out = np.zeros(3, np.float64)
        tot = ctypes.c_uint64()
        self._check(self.lib.evsim_ref_events_per_pixel_second(_ptr(ev), _i64(len(ev)), _i32(w), _i32(h),
                                                               ctypes.c_double(duration), _ptr(out),
                                                               ctypes.byref(tot)))
        return float(out[0]), float(out[1]), float(out[2]), int(tot.value)

    def accumulate(self, events: np.ndarray, w: int, h: int, t0: int, t1: int) -> np.ndarray:
        ev = self._ev24(events)
        out = np.zeros((h, w), np.uint8)
        self._check(self.lib.evsim_ref_accumulate(_ptr(ev), _i64(len(ev)), _i32(w), _i32(h), _i64(t0), _i64(t1),
                                                  _ptr(out)))
        return out
