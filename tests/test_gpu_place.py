"""Merged multi-GPU output on the device (-m gpu): each band's (or stream's)
events placed at its global offsets in one buffer (evsim_gpu_place_events),
offsets from per-(band, link) counts over the common link timeline
(parallel.timeline_counts / segment_dst_offsets) — SURVEY.md §8e.  The merged
buffer must equal the whole-frame stream (event order (t, y, x, p),
include/evsim/types.hpp:64-69).

The two-process test maps rank 0's buffer into rank 1 with CUDA IPC
(evsim_gpu_ipc_handle / evsim_gpu_ipc_open) — the path the ranks of a
multi-GPU run take over NVLink — on the one GPU available here (no kernel of
one process waits on the other's)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from paper_2209_04634_b200 import Simulator, SimulatorConfig, scenes
from paper_2209_04634_b200.abi import Method, make_config
from paper_2209_04634_b200.parallel import (band_rows, link_timeline, segment_dst_offsets, shard_streams,
                                            timeline_counts)

pytestmark = pytest.mark.gpu


def _segs(ev):
    S = int(ev.n_segments)
    seg_t = np.ctypeslib.as_array(ev.seg_t, shape=(S,)).copy() if S else np.zeros(0, np.int64)
    seg_off = np.ctypeslib.as_array(ev.seg_offset, shape=(S + 1,)).copy()
    return seg_t, seg_off


def _cfg(mode):
    return make_config(Method.dense, n_interp=8, contrast_mode=mode, c_pos_log=0.1, c_neg_log=-0.1)


@pytest.mark.parametrize("bands", [2, 3])
@pytest.mark.parametrize("mode", [0, 1])
def test_bands_placed_into_one_buffer_equal_whole_frame(bands, mode):
    import torch
    frames, ts = scenes.generate("c5", n_frames=6, width=200, height=150)
    frames = frames.copy()
    frames[:, 100:, :] = 90  # a static lower region: some bands miss some links
    frames[4, 120, 10] = 240
    cfg = _cfg(mode)
    full = Simulator(SimulatorConfig.from_c(cfg))
    exp = full.push_frames(frames, ts).events
    d = torch.from_numpy(frames).cuda()
    sims = []
    for r in range(bands):
        s = Simulator(SimulatorConfig.from_c(cfg))
        s.set_row_band(*band_rows(150, bands, r))
        sims.append(s)
    timeline = link_timeline(ts, 8)
    outs = [s.push_frames_device(d.data_ptr(), len(frames), 200, 150, ts) for s in sims]
    tabs = [_segs(e) for e in outs]
    counts = np.stack([timeline_counts(t, o, timeline) for t, o in tabs])
    merged = torch.zeros(int(counts.sum()), dtype=torch.int32, device="cuda")
    for r, (s, (seg_t, _)) in enumerate(zip(sims, tabs)):
        s.place_events(merged.data_ptr(), segment_dst_offsets(counts, r, timeline, seg_t))
    torch.cuda.synchronize()
    packed = merged.cpu().numpy().view(np.uint32)
    assert len(packed) == len(exp)
    assert np.array_equal(packed & 0xFFFF, exp["x"]) and np.array_equal((packed >> 16) & 0x7FFF, exp["y"])
    assert np.array_equal(np.where(packed >> 31, -1, 1), exp["p"])


def test_streams_placed_stream_major():
    """Independent streams (c4's sharding): stream-major merged output."""
    import torch
    cfg = _cfg(1)
    datas = [scenes.generate("c4", n_frames=4, stream=k, width=96, height=64) for k in range(3)]
    outs, sims = [], []
    for f, t in datas:
        s = Simulator(SimulatorConfig.from_c(cfg))
        outs.append(s.push_frames(f, t).events)
        sims.append(s)
    n = [len(o) for o in outs]
    merged = torch.zeros(sum(n), dtype=torch.int32, device="cuda")
    base = 0
    for k, (s, (f, t)) in enumerate(zip(sims, datas)):
        s.reset()
        d = torch.from_numpy(f).cuda()
        ev = s.push_frames_device(d.data_ptr(), len(f), 96, 64, t)
        seg_t, seg_off = _segs(ev)
        s.place_events(merged.data_ptr(), base + seg_off[:-1])
        base += int(ev.n_events)
    torch.cuda.synchronize()
    got = merged.cpu().numpy().view(np.uint32)
    exp = np.concatenate([o["x"].astype(np.uint32) | (o["y"].astype(np.uint32) << 16) |
                          np.where(o["p"] < 0, 0x80000000, 0).astype(np.uint32) for o in outs])
    assert np.array_equal(got, exp)
    assert list(shard_streams(3, 2, 0)) == [0, 1]


def _ipc_worker(rank, q_handle, q_done, q_result):
    import torch
    torch.cuda.set_device(0)
    from paper_2209_04634_b200.parallel import close_shared, open_shared, share_buffer
    frames, ts = scenes.generate("c5", n_frames=5, width=160, height=120)
    cfg = _cfg(1)
    sim = Simulator(SimulatorConfig.from_c(cfg))
    sim.set_row_band(*band_rows(120, 2, rank))
    d = torch.from_numpy(frames).cuda()
    ev = sim.push_frames_device(d.data_ptr(), len(frames), 160, 120, ts)
    timeline = link_timeline(ts, 8)
    seg_t, seg_off = _segs(ev)
    mine = timeline_counts(seg_t, seg_off, timeline)
    q_result.put(("counts", rank, mine))
    all_counts = q_handle.get()  # rank 0 relays the gathered counts (stands in for the all-gather)
    if rank == 0:
        total = int(all_counts.sum())
        buf = torch.zeros(total, dtype=torch.int32, device="cuda")
        q_result.put(("handle", 0, share_buffer(buf.data_ptr())))
        dst = buf.data_ptr()
    else:
        handle = q_handle.get()
        dst = open_shared(handle, 0)
    sim.place_events(dst, segment_dst_offsets(all_counts, rank, timeline, seg_t))
    torch.cuda.synchronize()
    q_result.put(("placed", rank, None))
    q_done.get()
    if rank == 0:
        q_result.put(("merged", 0, buf.cpu().numpy().view(np.uint32).copy()))
    else:
        close_shared(dst, 0)
    q_done.get()


def test_ipc_placement_two_processes():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    qh = [ctx.Queue(), ctx.Queue()]
    qd = [ctx.Queue(), ctx.Queue()]
    qr = ctx.Queue()
    ps = [ctx.Process(target=_ipc_worker, args=(r, qh[r], qd[r], qr)) for r in range(2)]
    for p in ps:
        p.start()
    counts = {}
    while len(counts) < 2:
        kind, r, v = qr.get(timeout=300)
        counts[r] = v
    all_counts = np.stack([counts[0], counts[1]])
    for r in range(2):
        qh[r].put(all_counts)
    kind, _, handle = qr.get(timeout=300)
    assert kind == "handle"
    qh[1].put(handle)
    placed = 0
    while placed < 2:
        kind, r, _ = qr.get(timeout=300)
        placed += kind == "placed"
    for r in range(2):
        qd[r].put(1)
    kind, _, merged = qr.get(timeout=300)
    for r in range(2):
        qd[r].put(1)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    frames, ts = scenes.generate("c5", n_frames=5, width=160, height=120)
    exp = Simulator(SimulatorConfig.from_c(_cfg(1))).push_frames(frames, ts).events
    assert len(merged) == len(exp)
    assert np.array_equal(merged & 0xFFFF, exp["x"]) and np.array_equal((merged >> 16) & 0x7FFF, exp["y"])
    assert np.array_equal(np.where(merged >> 31, -1, 1), exp["p"])
