"""Order-sensitive 64-bit checksum of one frame's event stream.

Used to pin whole timed sequences (tests/golden/sequences.json, made from the
compiled reference by tests/golden/make_sequences.py) against the device
output without shipping gigabytes of events.  For the events j = 0..n-1 of
one input frame (the events a push_frame call returns, in the reference's
order (t, y, x, p), src/simulate.cpp:36-40):

    v_j = x | y << 16 | (p < 0) << 31 | (t_j - t_prev) << 32      (u64)
    h   = sum_j splitmix64(v_j + j * 0x9E3779B97F4A7C15)          (mod 2^64)

t_prev is the previous frame's timestamp (every event of the frame lies in
(t_prev, t_frame]).  The same function is evaluated on packed device records
(bits 0-15 x, 16-30 y, 31 = negative) with torch, on the GPU, so bench.py can
check its own output without a device-to-host copy of the events.
"""
from __future__ import annotations

import numpy as np

GOLD = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB


def _s64(c: int) -> int:
    return c - (1 << 64) if c >= (1 << 63) else c


def _mix_np(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(M1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(M2)
    return z ^ (z >> np.uint64(31))


def frame_hash_np(x, y, t, p, t_prev: int, chunk: int = 1 << 24) -> int:
    """Checksum of one frame's events given as columns (numpy)."""
    n = len(x)
    h = np.uint64(0)
    with np.errstate(over="ignore"):
        for a in range(0, n, chunk):
            b = min(n, a + chunk)
            v = (np.asarray(x[a:b], np.uint64) | (np.asarray(y[a:b], np.uint64) << np.uint64(16))
                 | ((np.asarray(p[a:b]) < 0).astype(np.uint64) << np.uint64(31))
                 | ((np.asarray(t[a:b], np.int64) - np.int64(t_prev)).astype(np.uint64) << np.uint64(32)))
            j = np.arange(a, b, dtype=np.uint64)
            h = h + _mix_np(v + j * np.uint64(GOLD)).sum(dtype=np.uint64)
    return int(h)


def frame_hash_packed_np(packed: np.ndarray, seg_t: np.ndarray, seg_off: np.ndarray, t_prev: int) -> int:
    """Checksum from packed records + their segment table (numpy)."""
    packed = np.asarray(packed, np.uint32)
    t = np.repeat(np.asarray(seg_t, np.int64), np.diff(np.asarray(seg_off, np.int64)))
    x = packed & np.uint32(0xFFFF)
    y = (packed >> np.uint32(16)) & np.uint32(0x7FFF)
    p = np.where(packed >> np.uint32(31), -1, 1)
    return frame_hash_np(x, y, t, p, t_prev)


# ---------------------------------------------------------------- torch (device)

def _lshr(z, s: int):
    import torch
    return (z >> s) & ((1 << (64 - s)) - 1)


def _mix_torch(z):
    z = (z ^ _lshr(z, 30)) * _s64(M1)
    z = (z ^ _lshr(z, 27)) * _s64(M2)
    return z ^ _lshr(z, 31)


def frame_hash_packed_torch(packed_i32, seg_dt, seg_len, seg_jbase=None, chunk: int = 1 << 25) -> int:
    """Partial checksum of packed device records: `packed_i32` (int32 CUDA
    tensor) holds consecutive segments of one frame, segment s with
    seg_len[s] events at timestamp t_prev + seg_dt[s]; its events have frame
    indices j = seg_jbase[s] + 0, 1, ... (default: contiguous from 0).  The
    terms of disjoint event sets add (mod 2^64), so row bands sum their
    partial checksums.  int64 arithmetic wraps like u64."""
    import torch
    dev = packed_i32.device
    seg_dt = np.asarray(seg_dt, np.int64)
    seg_len = np.asarray(seg_len, np.int64)
    starts = np.concatenate([[0], np.cumsum(seg_len)[:-1]]).astype(np.int64)
    if seg_jbase is None:
        seg_jbase = starts
    seg_jbase = np.asarray(seg_jbase, np.int64)
    n = int(seg_len.sum())
    total = torch.zeros((), dtype=torch.int64, device=dev)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        s0 = int(np.searchsorted(starts, a, side="right") - 1)
        s1 = int(np.searchsorted(starts, b - 1, side="right") - 1)
        lens = np.minimum(starts[s0:s1 + 1] + seg_len[s0:s1 + 1], b) - np.maximum(starts[s0:s1 + 1], a)
        rep = torch.from_numpy(lens).to(dev)
        dt = torch.repeat_interleave(torch.from_numpy(seg_dt[s0:s1 + 1]).to(dev), rep, output_size=b - a)
        # j = jbase[s] + (i - start[s]) for event i of segment s
        shift = torch.repeat_interleave(torch.from_numpy(seg_jbase[s0:s1 + 1] - starts[s0:s1 + 1]).to(dev), rep,
                                        output_size=b - a)
        v = (packed_i32[a:b].to(torch.int64) & 0xFFFFFFFF) | (dt << 32)
        j = torch.arange(a, b, dtype=torch.int64, device=dev) + shift
        total += _mix_torch(v + j * _s64(GOLD)).sum()
    return int(total.item()) & ((1 << 64) - 1)


def device_int32(ptr: int, n: int, device: int):
    """An int32 CUDA tensor viewing n records at device address ptr (no copy)."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (int(n),), "typestr": "<i4", "data": (int(ptr), False), "version": 2}

    if n == 0:
        return torch.zeros(0, dtype=torch.int32, device=f"cuda:{device}")
    return torch.as_tensor(_View(), device=f"cuda:{device}")


def push_frame_hashes(d_packed: int, seg_t, seg_off, frame_ts, device: int, timeline=None, jbase=None) -> list:
    """Per-frame (count, checksum) of one push's device events.

    frame_ts: timestamps of the push's interval ends, preceded by the previous
    frame's (frame f covers (frame_ts[f], frame_ts[f+1]]).  seg_t / seg_off:
    the push's segment table (evsim_gpu_events).  Row bands: `timeline`
    (every link timestamp of the push, ascending) with `jbase` (per timeline
    entry, the frame index of this band's first event there) gives the
    band's partial checksums (see frame_hash_packed_torch)."""
    seg_t = np.asarray(seg_t, np.int64)
    seg_off = np.asarray(seg_off, np.int64)
    out = []
    for f in range(len(frame_ts) - 1):
        t0, t1 = int(frame_ts[f]), int(frame_ts[f + 1])
        a = int(np.searchsorted(seg_t, t0, side="right"))
        b = int(np.searchsorted(seg_t, t1, side="right"))
        lo, hi = int(seg_off[a]), int(seg_off[b])  # seg_off has len(seg_t) + 1 entries
        lens = seg_off[a + 1:b + 1] - seg_off[a:b]
        jb = None
        if timeline is not None:
            idx = np.searchsorted(np.asarray(timeline, np.int64), seg_t[a:b])
            jb = np.asarray(jbase, np.int64)[idx]
        view = device_int32(d_packed + 4 * lo, hi - lo, device)
        h = frame_hash_packed_torch(view, seg_t[a:b] - t0, lens, jb) if hi > lo else 0
        out.append((hi - lo, h))
    return out
