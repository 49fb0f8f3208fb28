"""The compact wire format (evsim_gpu_push_frames_wire + evsim_gpu_wire_unpack)
against the packed stream of the same push and the oracle (-m gpu).

The wire format carries the reference's event stream (std::vector<Event>,
include/evsim/types.hpp:54-80) as one plane bit per pixel-link plus one
polarity bit per event; unpacking must give exactly the events push_frames
returns (order (t, y, x, p), finalize's stable sort for equal timestamps,
src/simulate.cpp:36-40), in packed and in 24-byte form.
"""
from __future__ import annotations

import numpy as np
import pytest

from helpers import assert_same_events, concat, run_oracle_stream
from paper_2209_04634_b200 import Simulator, SimulatorConfig, scenes
from paper_2209_04634_b200.abi import Method, make_config, unpack_events

pytestmark = pytest.mark.gpu


def _both(cfg, frames, ts, chunk=0, band=None):
    a = Simulator(SimulatorConfig.from_c(cfg))
    b = Simulator(SimulatorConfig.from_c(cfg))
    if band:
        a.set_row_band(*band)
        b.set_row_band(*band)
    exp = a.push_frames(frames, ts).events
    wire = b.push_frames_wire(frames, ts, chunk=chunk)
    return exp, wire


def _check(exp, wire):
    ev24 = wire.unpack(fmt=1)
    assert_same_events(ev24, exp)
    packed = wire.unpack(fmt=0, threads=3)
    seg_t, seg_off = wire.segments()
    assert_same_events(unpack_events(packed, seg_t, seg_off), exp)
    assert wire.n_events == len(exp)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("chunk", [0, 7])
def test_wire_dense_matches_packed(mode, chunk):
    frames, ts = scenes.generate("c2", n_frames=30, width=131, height=77)
    cfg = make_config(Method.dense, n_interp=10, contrast_mode=mode, c_pos_log=0.1, c_neg_log=-0.1)
    exp, wire = _both(cfg, frames, ts, chunk=chunk)
    assert len(exp) > 1000
    _check(exp, wire)


def test_wire_dense_c5_like_dense_events():
    """High density (unblurred noise + pan + flicker, like c5): most words
    carry events, polarity runs cross u32 words everywhere."""
    frames, ts = scenes.generate("c5", n_frames=9, width=300, height=170)
    cfg = make_config(Method.dense, n_interp=32, contrast_mode=1, c_pos_log=0.1, c_neg_log=-0.1)
    exp, wire = _both(cfg, frames, ts, chunk=4)
    assert len(exp) > 0.1 * 300 * 170 * 33 * 8
    _check(exp, wire)


def test_wire_collisions_merge_links(oracle):
    """dt < K: equal link timestamps form one segment ordered (y, x, p)."""
    frames, _ = scenes.generate("c1", n_frames=6, width=48, height=40)
    ts = np.array([0, 5, 9, 12, 100, 104], np.int64)
    for mode in (0, 1):
        cfg = make_config(Method.dense, n_interp=10, contrast_mode=mode, c_pos_log=0.05, c_neg_log=-0.05)
        exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
        _, wire = _both(cfg, frames, ts)
        assert_same_events(wire.unpack(fmt=1), exp)


@pytest.mark.parametrize("method,n", [(Method.difference_only, 0), (Method.sparse, 6)])
def test_wire_other_methods(method, n):
    frames, ts = scenes.generate("c3", n_frames=12, width=160, height=96)
    for mode in (0, 1):
        cfg = make_config(method, n_interp=n, contrast_mode=mode, c_pos_log=0.15, c_neg_log=-0.15)
        exp, wire = _both(cfg, frames, ts, chunk=5)
        _check(exp, wire)


def test_wire_no_endpoints_and_band():
    frames, ts = scenes.generate("c2", n_frames=10, width=96, height=80)
    cfg = make_config(Method.dense, n_interp=6, include_endpoints=0, contrast_mode=0)
    exp, wire = _both(cfg, frames, ts)
    _check(exp, wire)
    cfg = make_config(Method.dense, n_interp=6, contrast_mode=1, c_pos_log=0.1, c_neg_log=-0.1)
    exp, wire = _both(cfg, frames, ts, band=(17, 53))
    assert wire.c.row0 == 17 and wire.c.rows == 36
    _check(exp, wire)


def test_wire_rejects_small_buffers_and_magnitude():
    from paper_2209_04634_b200 import InvalidArgument
    from paper_2209_04634_b200.simulator import WireBuffer
    frames, ts = scenes.generate("c2", n_frames=4, width=64, height=48)
    cfg = make_config(Method.dense, n_interp=4, contrast_mode=0)
    sim = Simulator(SimulatorConfig.from_c(cfg))
    small = WireBuffer(2, 10, 10, pinned=False)
    with pytest.raises(InvalidArgument, match="too small"):
        sim.push_frames_wire(frames, ts, wire=small)
    mag = Simulator(SimulatorConfig.from_c(make_config(Method.dense, n_interp=4, events_per_crossing=1)))
    with pytest.raises(InvalidArgument, match="magnitude"):
        mag.push_frames_wire(frames, ts)


def test_wire_continues_a_stream():
    """State carries across calls: wire calls interleaved with packed pushes."""
    frames, ts = scenes.generate("c2", n_frames=20, width=80, height=64)
    cfg = make_config(Method.dense, n_interp=5, contrast_mode=1, c_pos_log=0.1, c_neg_log=-0.1)
    a = Simulator(SimulatorConfig.from_c(cfg))
    exp = a.push_frames(frames, ts).events
    b = Simulator(SimulatorConfig.from_c(cfg))
    parts = [b.push_frames(frames[:5], ts[:5]).events,
             b.push_frames_wire(frames[5:12], ts[5:12], chunk=3).unpack(fmt=1),
             b.push_frames(frames[12:15], ts[12:15]).events,
             b.push_frames_wire(frames[15:], ts[15:]).unpack(fmt=1)]
    assert_same_events(np.concatenate(parts), exp)


def test_wire_call_longer_than_a_launch():
    """A wire call may hold more frames than max_batch: its chunks are
    launches of <= max_batch pairs (events never need one device buffer)."""
    frames, ts = scenes.generate("c5", n_frames=21, width=1280, height=800)
    cfg = make_config(Method.dense, n_interp=32, contrast_mode=1, c_pos_log=0.1, c_neg_log=-0.1)
    a = Simulator(SimulatorConfig.from_c(cfg))
    mb = a.max_batch(1280, 800)
    assert mb < 21
    exp = a.push_frames(frames, ts)  # (split into max_batch calls by the wrapper)
    b = Simulator(SimulatorConfig.from_c(cfg))
    wire = b.push_frames_wire(frames, ts)
    assert wire.n_events == len(exp.events)
    packed = wire.unpack(fmt=0)
    seg_t, seg_off = wire.segments()
    assert_same_events(unpack_events(packed, seg_t, seg_off), exp.events)
