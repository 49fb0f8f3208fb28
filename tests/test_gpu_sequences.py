"""Whole BASELINE sequences through the GPU path against the compiled
reference (-m gpu).

tests/golden/sequences.json holds, per (config, mode), every frame's event
count and order-sensitive checksum from the reference's own streaming
Simulator (tests/golden/make_sequences.py, oracle/_ref; src/simulate.cpp:306-347).
Here the same sequences run through

* the pipelined device push (evsim_gpu_push_frames, max batches: flow
  sub-batches, per-sub-batch emits, the flow / chain overlap) — checksums
  reduced on the device (paper_2209_04634_b200/seqhash.py);
* the streamed host call (evsim_gpu_push_frames_streamed: host frames in,
  host events out, chunked and overlapped) — checksums on the host;
* frame-by-frame pushes for the smaller configs.

Full sizes: c1 346x260 x64, c2 640x480 x128, c3 1280x720 x256, c4 stream 0
1920x1080 x120, c5 3840x2160 x60; both contrast modes; c2 also with the
high-quality flow preset (keys "c2:<mode>:hq").
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_2209_04634_b200 import scenes

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sequences.json")
SEQS = json.load(open(GOLDEN)) if os.path.exists(GOLDEN) else {}
KEYS = sorted(SEQS)

_frames_cache = {}


def _frames(name):
    if name not in _frames_cache:
        _frames_cache.clear()
        _frames_cache[name] = scenes.generate(scenes.CONFIGS[name], stream=0)
    return _frames_cache[name]


def _split(key):
    """(config, mode, preset) of a key "c2:log" / "c2:log:hq"."""
    return (tuple(key.split(":")) + ("lq",))[:3]


def _cfg(name, mode, preset="lq"):
    from paper_2209_04634_b200.abi import Method, make_config
    c = scenes.CONFIGS[name]
    cp, cn = scenes.LINEAR_THRESHOLDS[c.method]
    return make_config(Method[c.method], n_interp=c.n_interp, c_pos=cp, c_neg=cn,
                       contrast_mode=1 if mode == "log" else 0, c_pos_log=c.contrast, c_neg_log=-c.contrast,
                       flow_preset=1 if preset == "hq" else 0)


def test_golden_sequences_cover_every_config():
    """The committed checksums pin c1-c5 (c4: stream 0) in both modes, for the
    frames scenes.generate makes (the generator's output hash is recorded)."""
    want = [f"{c}:{m}" for c in ("c1", "c2", "c3", "c4", "c5") for m in ("log", "linear")]
    want += ["c2:log:hq", "c2:linear:hq"]  # the high-quality flow preset (types.hpp:93)
    assert sorted(SEQS) == sorted(want)
    for k, g in SEQS.items():
        assert len(g["counts"]) == g["n_frames"] == scenes.CONFIGS[g["config"]].n_frames, k
        assert g["counts"][0] == 0  # the warm-up frame emits nothing


@pytest.mark.parametrize("key", ["c1:log", "c1:linear", "c2:log", "c3:log"])
def test_generator_matches_pinned_frames(key):
    """scenes.generate reproduces the frames the checksums were made from."""
    import hashlib
    g = SEQS[key]
    frames, ts = _frames(g["config"])
    assert hashlib.sha256(np.ascontiguousarray(frames).tobytes()).hexdigest() == g["frames_sha256"]
    assert [int(t) for t in ts] == g["timestamps"]


def _check(key, got):
    g = SEQS[key]
    counts = [c for c, _ in got]
    hashes = [f"{h:016x}" for _, h in got]
    n = len(counts)
    bad = [i for i in range(n) if counts[i] != g["counts"][i + 1] or hashes[i] != g["hashes"][i + 1]]
    assert not bad, f"{key}: {len(bad)} of {n} frames differ, first frame {bad[0] + 1}: " \
                    f"{counts[bad[0]]} events vs {g['counts'][bad[0] + 1]}"


def _device_pass(name, mode, batch=0, preset="lq"):
    import torch

    from paper_2209_04634_b200 import Simulator, SimulatorConfig
    from paper_2209_04634_b200.seqhash import push_frame_hashes
    frames, ts = _frames(name)
    c = scenes.CONFIGS[name]
    sim = Simulator(SimulatorConfig.from_c(_cfg(name, mode, preset)))
    d = torch.from_numpy(frames).cuda()
    P = c.width * c.height
    mb = sim.max_batch(c.width, c.height)
    batch = min(batch or mb, mb)
    got = []
    for a in range(0, len(frames), batch):
        nb = min(batch, len(frames) - a)
        ev = sim.push_frames_device(d.data_ptr() + a * P, nb, c.width, c.height, ts[a:a + nb], on_device=True)
        S = int(ev.n_segments)
        seg_t = np.ctypeslib.as_array(ev.seg_t, shape=(S,)).copy() if S else np.zeros(0, np.int64)
        seg_off = np.ctypeslib.as_array(ev.seg_offset, shape=(S + 1,)).copy()
        f0 = max(a, 1)
        got += push_frame_hashes(int(ev.d_packed), seg_t, seg_off, ts[f0 - 1:a + nb], 0)
    sim.close()
    return got


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_sequence_pipelined_push_matches_reference(key):
    name, mode, preset = _split(key)
    _check(key, _device_pass(name, mode, preset=preset))


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["c2:log", "c2:linear", "c3:log", "c1:log", "c2:log:hq"])
def test_sequence_small_batches_match_reference(key):
    """Batches of 5 frames: a push boundary inside the sequence every 5
    frames (the state carried across pushes: ring, pyramids, log state)."""
    name, mode, preset = _split(key)
    _check(key, _device_pass(name, mode, batch=5, preset=preset))


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["c1:log", "c1:linear", "c2:log", "c2:linear", "c3:log", "c3:linear",
                                 "c2:linear:hq"])
def test_sequence_streamed_call_matches_reference(key):
    """Host frames in, host events out (evsim_gpu_push_frames_streamed)."""
    from paper_2209_04634_b200 import Simulator, SimulatorConfig
    from paper_2209_04634_b200.seqhash import frame_hash_packed_np
    name, mode, preset = _split(key)
    frames, ts = _frames(name)
    c = scenes.CONFIGS[name]
    sim = Simulator(SimulatorConfig.from_c(_cfg(name, mode, preset)))
    mb = sim.max_batch(c.width, c.height)
    got = []
    for a0 in range(0, len(frames), mb):  # calls of at most max_batch frames, chunks of 24 inside
        a1 = min(len(frames), a0 + mb)
        packed, seg_t, seg_off = sim.push_frames_streamed(frames[a0:a1], ts[a0:a1], chunk=24)
        for f in range(max(a0, 1), a1):
            a = int(np.searchsorted(seg_t, ts[f - 1], side="right"))
            b = int(np.searchsorted(seg_t, ts[f], side="right"))
            lo, hi = int(seg_off[a]), int(seg_off[b])
            got.append((hi - lo, frame_hash_packed_np(packed[lo:hi], seg_t[a:b], seg_off[a:b + 1] - lo,
                                                      int(ts[f - 1]))))
    sim.close()
    _check(key, got)
