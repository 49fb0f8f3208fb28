"""Multi-GPU sharding of the event-simulation path.

One process per GPU.  Two partitions, both without any data-path exchange:

* streams (config c4): rank r owns a contiguous block of camera streams and
  keeps their state (frame ring, pyramids, log state) resident; a merged
  output needs only each stream's event count -> ``merged_offsets``.
* row bands (config c5): every rank holds the full frame, builds the full
  pyramids locally, solves only the patch rows its band depends on
  (``band_plan``, the reference's own index math, exact for any preset) and
  emits the events of its rows.  Within one timestamp the reference orders
  events by (y, x), so the global stream is, per segment, band 0's events,
  then band 1's, ...: ``band_offsets`` from an all-gather of per-(band,
  segment) counts.

``gather_counts`` is the only collective (NCCL on GPU, gloo in the CPU tests).
"""
from __future__ import annotations

import dataclasses
from typing import Sequence

import numpy as np


# ----------------------------------------------------------------------------- streams

def shard_streams(n_streams: int, world_size: int, rank: int) -> range:
    """Contiguous block of streams owned by `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_streams, world_size)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def merged_offsets(counts: Sequence[int]) -> np.ndarray:
    """Exclusive prefix of per-stream event counts: where each stream's events
    start in a merged (stream-major) output."""
    c = np.asarray(counts, dtype=np.int64)
    return np.concatenate([[0], np.cumsum(c)[:-1]]) if len(c) else np.zeros(0, np.int64)


def gather_counts(local: Sequence[int], group=None, device=None) -> np.ndarray:
    """All-gather of equally sized int64 count vectors -> (world, len) array."""
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(np.asarray(local, dtype=np.int64), device=device)
    ws = dist.get_world_size(group)
    out = [torch.zeros_like(t) for _ in range(ws)]
    dist.all_gather(out, t, group=group)
    return np.stack([o.cpu().numpy() for o in out])


# ----------------------------------------------------------------------------- row bands

def band_rows(height: int, world_size: int, rank: int, align: int = 1) -> tuple[int, int]:
    """Event rows [y0, y1) of `rank`'s band (aligned cut points)."""
    cuts = [min(height, ((height * b // world_size) + align - 1) // align * align) for b in range(world_size)]
    cuts.append(height)
    cuts[0] = 0
    return cuts[rank], cuts[rank + 1]


def _patch_centers(extent: int, radius: int, stride: int) -> list[int]:
    # flow.cpp:97-107
    if extent <= 2 * radius + 1:
        return [(extent - 1) // 2]
    last = extent - 1 - radius
    c = list(range(radius, last + 1, stride))
    if c[-1] != last:
        c.append(last)
    return c


def _interp_idx(centers: list[int], extent: int) -> list[int]:
    # interp_table's idx (flow.cpp:111-128)
    idx = [0] * extent
    if len(centers) < 2:
        return idx
    j = 0
    for x in range(extent):
        if x <= centers[0]:
            continue
        if x >= centers[-1]:
            idx[x] = len(centers) - 2
            continue
        while j + 2 < len(centers) and centers[j + 1] <= x:
            j += 1
        idx[x] = j
    return idx


def _effective_levels(requested: int, w: int, h: int) -> int:
    levels = max(1, requested)
    while levels > 1 and (min(w, h) >> (levels - 1)) < 8:
        levels -= 1
    return levels


@dataclasses.dataclass
class BandPlan:
    rows: tuple[int, int]                  # event rows [y0, y1) at level 0
    patch_rows: list[tuple[int, int]]      # per level l: patch-row range [j0, j1) to solve
    level_heights: list[int]


def band_plan(width: int, height: int, rows: tuple[int, int], levels: int = 3, radius: int = 4) -> BandPlan:
    """Patch rows each pyramid level must solve so that the level-0 flow at
    event rows [y0, y1) is bit-identical to the full-frame solve.

    Level 0: densification reads patch rows iy[y] and iy[y]+1 (flow.cpp:224-245).
    Level l+1: the seed of every needed level-l patch centre cy samples the
    densified level-(l+1) field at sy = (cy + 0.5) * ry - 0.5 (flow.cpp:130-147),
    i.e. rows trunc(clamp(sy)) and +1, whose densification reads patch rows
    iy'[row] and +1.  Solving a patch reads only the (full, replicated) level
    images, so these rows are the complete dependency set.
    """
    L = _effective_levels(levels, width, height)
    hs = [height]
    for _ in range(1, L):
        hs.append((hs[-1] + 1) // 2)
    stride = max(1, radius)
    centers = [_patch_centers(hl, radius, stride) for hl in hs]
    idx = [_interp_idx(c, hl) for c, hl in zip(centers, hs)]
    y0, y1 = rows
    need = [set() for _ in range(L)]
    for y in range(y0, y1):
        j = idx[0][y]
        need[0].update({min(j, len(centers[0]) - 1), min(j + 1, len(centers[0]) - 1)})
    for l in range(L - 1):
        hf, hc = hs[l], hs[l + 1]
        ry = np.float32(hc) / np.float32(hf)
        for j in need[l]:
            cy = centers[l][j]
            sy = np.float32((np.float32(cy) + np.float32(0.5)) * ry - np.float32(0.5))
            sy = min(max(float(sy), 0.0), float(hc - 1))
            r0 = int(sy)
            for rr in (r0, min(r0 + 1, hc - 1)):
                jj = idx[l + 1][rr]
                need[l + 1].update({min(jj, len(centers[l + 1]) - 1), min(jj + 1, len(centers[l + 1]) - 1)})
    patch_rows = [(min(n), max(n) + 1) if n else (0, 0) for n in need]
    return BandPlan(rows=(y0, y1), patch_rows=patch_rows, level_heights=hs)


def band_input_halo(plan: BandPlan, radius: int) -> int:
    """Rows of level-0 input above/below the band the planned patches touch
    through their templates (before flow displacement) — the part of the
    frame a band-local (non-replicated) implementation would need."""
    y0, y1 = plan.rows
    lo = hi = 0
    h0 = plan.level_heights[0]
    for l, (j0, j1) in enumerate(plan.patch_rows):
        centers = _patch_centers(plan.level_heights[l], radius, max(1, radius))
        if j1 <= j0:
            continue
        scale = 1 << l
        top = (centers[j0] - radius - 1) * scale
        bot = (centers[j1 - 1] + radius + 2) * scale
        lo = max(lo, y0 - max(0, top))
        hi = max(hi, min(h0, bot) - y1)
    return max(lo, hi)


def link_timeline(ts: Sequence[int], n_interp: int, include_endpoints: bool = True) -> np.ndarray:
    """Every distinct link timestamp of a push over frames ts (dense / sparse /
    difference_only chains: chain_pipeline, simulate.cpp:57-69, with
    sub_interval_end, simulate.hpp:15-19), ascending.  Every rank derives the
    same timeline from the timestamps alone, so per-band counts over it line
    up even where a band has no events (the device reports only the segments
    that hold events)."""
    K = n_interp + 1
    out = []
    for i in range(len(ts) - 1):
        t0, t1 = int(ts[i]), int(ts[i + 1])
        ks = range(1, K + 1) if include_endpoints or n_interp == 0 else range(2, K)
        for k in ks:
            out.append(t1 if k == K else t0 + (k * (t1 - t0) + K - 1) // K)
    return np.unique(np.asarray(out, np.int64))


def timeline_counts(seg_t: Sequence[int], seg_off: Sequence[int], timeline: np.ndarray) -> np.ndarray:
    """Events per timeline entry from a push's segment table (seg_t: the
    non-empty segments' timestamps, seg_off: their offsets + total); 0 where
    the band has no segment.  The vector every rank all-gathers."""
    seg_t = np.asarray(seg_t, np.int64)
    out = np.zeros(len(timeline), np.int64)
    if len(seg_t):
        idx = np.searchsorted(timeline, seg_t)
        if np.any(idx >= len(timeline)) or np.any(timeline[np.minimum(idx, len(timeline) - 1)] != seg_t):
            raise ValueError("timeline_counts: a segment timestamp is not on the timeline")
        out[idx] = np.diff(np.asarray(seg_off, np.int64))
    return out


def band_offsets(seg_counts: np.ndarray, rank: int) -> np.ndarray:
    """Output offsets of `rank`'s events per segment in the merged stream.

    seg_counts: (world, S) events per (band, segment) from gather_counts.
    Merged order = segment-major, band-minor (time, then rows)."""
    c = np.asarray(seg_counts, dtype=np.int64)
    seg_tot = c.sum(axis=0)
    seg_base = np.concatenate([[0], np.cumsum(seg_tot)[:-1]])
    before = c[:rank].sum(axis=0) if rank > 0 else np.zeros(c.shape[1], np.int64)
    return seg_base + before


def merge_band_events(band_events: Sequence[np.ndarray], seg_counts: np.ndarray) -> np.ndarray:
    """Assemble the global stream from each band's events (each band's
    events are in segment order) using band_offsets — what the ranks do with
    P2P writes into one buffer."""
    from .abi import EVENT_DTYPE
    c = np.asarray(seg_counts, dtype=np.int64)
    total = int(c.sum())
    out = np.zeros(total, EVENT_DTYPE)
    for r, ev in enumerate(band_events):
        offs = band_offsets(c, r)
        pos = 0
        for s in range(c.shape[1]):
            n = int(c[r, s])
            out[offs[s]:offs[s] + n] = ev[pos:pos + n]
            pos += n
    return out


# ----------------------------------------------------------------------------- merged output on the device

def segment_dst_offsets(all_counts: np.ndarray, rank: int, timeline: np.ndarray, seg_t: Sequence[int],
                        base: int = 0) -> np.ndarray:
    """Where this rank's non-empty segments (seg_t) go in the merged stream:
    all_counts is the (world, len(timeline)) all-gather of timeline_counts;
    merged order = timestamp-major, band (or stream) minor."""
    offs = band_offsets(all_counts, rank) + int(base)
    idx = np.searchsorted(timeline, np.asarray(seg_t, np.int64))
    return offs[idx].astype(np.int64)


def share_buffer(ptr: int) -> bytes:
    """64-byte CUDA IPC handle of a device allocation (evsim_gpu_ipc_handle),
    to broadcast to the other ranks."""
    import ctypes

    from . import _lib
    h = (ctypes.c_char * 64)()
    _lib.check(_lib.load().evsim_gpu_ipc_handle(ctypes.c_void_p(ptr), h))
    return bytes(h)


def open_shared(handle: bytes, device: int) -> int:
    """Map a peer process's buffer (share_buffer) into this one: its device
    address here (evsim_gpu_ipc_open, lazy peer access)."""
    import ctypes

    from . import _lib
    out = ctypes.c_void_p()
    h = (ctypes.c_char * 64).from_buffer_copy(handle)
    _lib.check(_lib.load().evsim_gpu_ipc_open(device, h, ctypes.byref(out)))
    return int(out.value)


def close_shared(ptr: int, device: int) -> None:
    import ctypes

    from . import _lib
    _lib.check(_lib.load().evsim_gpu_ipc_close(device, ctypes.c_void_p(ptr)))


# --------------------------------------------------------------------------- stacked streams

def stack_streams(frames: Sequence[np.ndarray]) -> np.ndarray:
    """S streams of (n, h, w) frames -> (n, S*h, w): frame k of the stack is
    stream 0's frame k on rows [0, h), stream 1's on [h, 2h), ...

    For difference_only (no flow, every pixel its own chain,
    simulate.cpp:322-327 -> core.cpp:5-46) one simulator over the stacked frame
    IS S independent simulators: the per-pixel rule never looks at a
    neighbour, and within one timestamp the reference orders events by
    (y, x) (types.hpp:64-69), so each segment of the stacked stream is
    stream 0's events, then stream 1's, ... — the same structure as row bands.
    All streams must share their timestamps.  This turns S small streams into
    one launch sequence (the batched c1 workload)."""
    arr = np.stack([np.asarray(f, np.uint8) for f in frames], axis=1)  # (n, S, h, w)
    n, S, h, w = arr.shape
    return np.ascontiguousarray(arr.reshape(n, S * h, w))


def split_stacked(packed: np.ndarray, seg_t: np.ndarray, seg_off: np.ndarray, n_streams: int, height: int) -> list:
    """The stacked stream's packed records (bits 0-15 x, 16-30 y, 31 negative)
    and segment table -> per stream (packed records with y - s*height, seg_t,
    seg_off).  Within a segment the records are ordered by y, so stream s's
    records are the run with s*height <= y < (s+1)*height."""
    packed = np.asarray(packed, np.uint32)
    seg_off = np.asarray(seg_off, np.int64)
    y = (packed >> np.uint32(16)) & np.uint32(0x7FFF)
    stream = (y // np.uint32(height)).astype(np.int64)
    out = []
    S = len(seg_t)
    # per segment, the boundaries of each stream's run (searchsorted on the
    # nondecreasing stream index inside the segment)
    bounds = np.zeros((S, n_streams + 1), np.int64)
    for k in range(S):
        a, b = int(seg_off[k]), int(seg_off[k + 1])
        bounds[k] = a + np.searchsorted(stream[a:b], np.arange(n_streams + 1), side="left")
    for s in range(n_streams):
        idx = np.concatenate([np.arange(bounds[k, s], bounds[k, s + 1]) for k in range(S)]) if S else np.zeros(0, int)
        rec = packed[idx].copy()
        rec = (rec & np.uint32(0x8000FFFF)) | (((y[idx] - np.uint32(s * height)) & np.uint32(0x7FFF)) << np.uint32(16))
        counts = bounds[:, s + 1] - bounds[:, s]
        keep = counts > 0
        off = np.concatenate([[0], np.cumsum(counts[keep])]).astype(np.int64)
        out.append((rec, np.asarray(seg_t, np.int64)[keep], off))
    return out
