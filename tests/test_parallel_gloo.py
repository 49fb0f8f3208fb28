"""CPU: the multi-GPU host logic with world_size 2 over gloo.

* streams: each rank simulates its own streams (oracle stands in for the
  device), event counts are all-gathered, merged offsets place every stream;
* row bands: each rank emits the events of its rows, per-(band, segment)
  counts are all-gathered, the merged stream equals the full-frame stream;
* band plan: the patch rows a band solves are the complete dependency set of
  its level-0 flow (perturbing everything else leaves it bit-identical).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2209_04634_b200.parallel import (band_offsets, band_plan, band_rows, merge_band_events, merged_offsets,
                                            shard_streams)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _stream_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from oracle import Oracle
    from paper_2209_04634_b200 import scenes
    from paper_2209_04634_b200.abi import Method, make_config
    from paper_2209_04634_b200.parallel import gather_counts

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_streams = 5
    mine = shard_streams(n_streams, world, rank)
    cfg = make_config(Method.dense, n_interp=3, contrast_mode=1, c_pos_log=0.15, c_neg_log=-0.15)
    counts = np.zeros(n_streams, np.int64)
    ora = Oracle()
    for s in mine:
        frames, ts = scenes.generate("c4", n_frames=3, stream=s, width=48, height=32)
        sim = ora.simulator(cfg)
        counts[s] = sum(len(sim.push_frame(frames[k], ts[k])) for k in range(3))
    all_counts = gather_counts(counts).sum(axis=0)  # each stream counted by its owner only
    np.save(os.path.join(out_dir, f"counts_{rank}.npy"), all_counts)
    dist.destroy_process_group()


def _band_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from oracle import Oracle
    from paper_2209_04634_b200 import scenes
    from paper_2209_04634_b200.abi import Method, make_config
    from paper_2209_04634_b200.parallel import gather_counts, link_timeline, timeline_counts

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    frames, ts = scenes.generate("c5", n_frames=3, width=96, height=64)
    frames = frames.copy()
    frames[:, 8:, :] = 128  # texture in the top rows only: band 1 is static ...
    frames[2, 50, 7] = 250  # ... but for one pixel in the last frame (events on some links only)
    cfg = make_config(Method.dense, n_interp=6, contrast_mode=1, c_pos_log=0.1, c_neg_log=-0.1)
    sim = Oracle().simulator(cfg)
    sim.push_frame(frames[0], ts[0])
    full = np.concatenate([sim.push_frame(frames[1], ts[1]), sim.push_frame(frames[2], ts[2])])
    y0, y1 = band_rows(64, world, rank)
    mine = full[(full["y"] >= y0) & (full["y"] < y1)]  # this band's device output (rows [y0, y1))
    # what a band handle reports: only the segments that hold events, so the
    # bands' segment tables differ in length; counts go over the common
    # link timeline every rank derives from the timestamps
    seg_t, first = np.unique(mine["t"], return_index=True)
    seg_off = np.append(first, len(mine))
    timeline = link_timeline(ts, 6)
    local = timeline_counts(seg_t, seg_off, timeline)
    counts = gather_counts(local)
    np.save(os.path.join(out_dir, f"nseg_{rank}.npy"), np.array([len(seg_t)]))
    # where evsim_gpu_place_events puts this band's segments in rank 0's buffer
    from paper_2209_04634_b200.parallel import segment_dst_offsets
    np.save(os.path.join(out_dir, f"dst_{rank}.npy"), segment_dst_offsets(counts, rank, timeline, seg_t))
    np.save(os.path.join(out_dir, f"segoff_{rank}.npy"), seg_off)
    np.save(os.path.join(out_dir, f"band_{rank}.npy"), mine)
    np.save(os.path.join(out_dir, f"bandcounts_{rank}.npy"), counts)
    if rank == 0:
        np.save(os.path.join(out_dir, "full.npy"), full)
    dist.destroy_process_group()


def _spawn(fn, tmp_path):
    mp.start_processes(fn, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True, start_method="spawn")


def test_shard_streams_cover_all():
    for n in (1, 5, 32):
        for ws in (1, 2, 3, 8):
            got = [list(shard_streams(n, ws, r)) for r in range(ws)]
            assert sum(got, []) == list(range(n))


def test_streams_gloo_world2(tmp_path):
    _spawn(_stream_worker, tmp_path)
    c0 = np.load(tmp_path / "counts_0.npy")
    c1 = np.load(tmp_path / "counts_1.npy")
    assert np.array_equal(c0, c1) and (c0 > 0).all()
    offs = merged_offsets(c0)
    assert offs[0] == 0 and np.array_equal(np.diff(offs), c0[:-1])


def test_row_bands_gloo_world2(tmp_path):
    _spawn(_band_worker, tmp_path)
    full = np.load(tmp_path / "full.npy")
    bands = [np.load(tmp_path / f"band_{r}.npy") for r in range(2)]
    counts = np.load(tmp_path / "bandcounts_0.npy")
    assert np.array_equal(counts, np.load(tmp_path / "bandcounts_1.npy"))
    n0, n1 = (int(np.load(tmp_path / f"nseg_{r}.npy")[0]) for r in range(2))
    assert n0 != n1  # the bands' own segment tables differ in length
    merged = merge_band_events(bands, counts)
    # the device placement's arithmetic: each band's segment s at dst[s]
    placed = np.zeros(len(full), full.dtype)
    for r in range(2):
        dst = np.load(tmp_path / f"dst_{r}.npy")
        off = np.load(tmp_path / f"segoff_{r}.npy")
        for q in range(len(dst)):
            placed[dst[q]:dst[q] + off[q + 1] - off[q]] = bands[r][off[q]:off[q + 1]]
    for f in ("x", "y", "t", "p"):
        assert np.array_equal(placed[f], full[f])
    for f in ("x", "y", "t", "p"):
        assert np.array_equal(merged[f], full[f])
    assert band_offsets(counts, 0)[0] == 0


def test_band_plan_is_complete_dependency_set(oracle):
    """lq: the flow at band rows depends only on a bounded neighbourhood —
    the planned patch rows' templates plus the flow displacement (SURVEY.md
    §8e: <= 56 level-0 px for lq).  Perturbing every row outside that
    neighbourhood leaves the band's flow bit-identical."""
    from paper_2209_04634_b200 import scenes
    from paper_2209_04634_b200.parallel import band_input_halo
    H, rows = 640, (288, 352)
    frames, _ = scenes.generate("c2", n_frames=2, width=96, height=H)
    a, b = frames[0], frames[1]
    du, dv = oracle.dense_flow(a, b, 3, 2, 4)
    plan = band_plan(96, H, rows, 3, 4)
    assert plan.patch_rows[0][0] > 0 and plan.patch_rows[0][1] < len(range(4, H - 4, 4)) + 1
    reach = band_input_halo(plan, 4) + 64  # templates + displacement bound
    lo, hi = rows[0] - reach, rows[1] + reach
    assert lo > 0 and hi < H
    a2, b2 = a.copy(), b.copy()
    rng = np.random.default_rng(1)
    a2[:lo] = rng.integers(0, 256, a2[:lo].shape)
    b2[:lo] = rng.integers(0, 256, b2[:lo].shape)
    a2[hi:] = rng.integers(0, 256, a2[hi:].shape)
    b2[hi:] = rng.integers(0, 256, b2[hi:].shape)
    du2, dv2 = oracle.dense_flow(a2, b2, 3, 2, 4)
    y0, y1 = rows
    assert np.array_equal(du[y0:y1].view(np.uint32), du2[y0:y1].view(np.uint32))
    assert np.array_equal(dv[y0:y1].view(np.uint32), dv2[y0:y1].view(np.uint32))
    # ... while the perturbation does change the flow elsewhere (the test bites)
    assert not np.array_equal(du, du2)


def test_band_plan_c5_halo_bounds():
    """for lq at 3840x2160 a 96-row halo suffices for G = 2/4/8."""
    from paper_2209_04634_b200.parallel import band_input_halo
    for G in (2, 4, 8):
        for r in range(G):
            rows = band_rows(2160, G, r, align=4)
            plan = band_plan(3840, 2160, rows, 3, 4)
            assert band_input_halo(plan, 4) <= 96
