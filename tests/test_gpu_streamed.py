"""GPU: evsim_gpu_push_frames_streamed (host frames in, host events out, with
upload / compute / download overlapped across chunks) returns exactly the
events of the reference's frame-by-frame Simulator::push_frame, for every
method / mode and chunking, and keeps the stream state consistent for later
pushes."""
import ctypes

import numpy as np
import pytest

from helpers import assert_same_events, concat, run_oracle_stream
from paper_2209_04634_b200 import Frame, InvalidArgument, SimulatorConfig, Simulator, scenes
from paper_2209_04634_b200.abi import EVENT_DTYPE, Method, make_config, unpack_events

pytestmark = pytest.mark.gpu


def _cfg(m, mode, incl=1):
    return make_config(m, n_interp=5 if m != Method.difference_only else 0, contrast_mode=mode,
                       include_endpoints=incl, c_pos_log=0.1, c_neg_log=-0.12, selection_threshold=4)


@pytest.mark.parametrize("m,mode,incl", [(Method.dense, 1, 1), (Method.dense, 0, 1), (Method.dense, 1, 0),
                                         (Method.sparse, 1, 1), (Method.sparse, 0, 0),
                                         (Method.difference_only, 0, 1), (Method.difference_only, 1, 1)])
@pytest.mark.parametrize("chunk", [0, 1, 3, 4])
def test_streamed_matches_oracle(oracle, m, mode, incl, chunk):
    frames, ts = scenes.generate("c2", n_frames=11, width=100, height=76)
    cfg = _cfg(m, mode, incl)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    packed, seg_t, seg_off = sim.push_frames_streamed(frames, ts, chunk=chunk)
    assert seg_off[-1] == packed.size
    assert_same_events(unpack_events(packed, seg_t, seg_off), exp)


def test_streamed_continues_stream_and_mixes_with_pushes(oracle):
    frames, ts = scenes.generate("c2", n_frames=14, width=80, height=64)
    cfg = _cfg(Method.dense, 1)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    got = [sim.push_frame(Frame.from_array(frames[0], ts[0])).events]
    p, t, o = sim.push_frames_streamed(frames[1:6], ts[1:6], chunk=2)
    got.append(unpack_events(p, t, o))
    got.append(sim.push_frames(frames[6:9], ts[6:9]).events)
    p, t, o = sim.push_frames_streamed(frames[9:14], ts[9:14], chunk=5)
    got.append(unpack_events(p, t, o))
    assert_same_events(concat(got), exp)


def test_streamed_small_destination_keeps_events_on_device(oracle):
    frames, ts = scenes.generate("c2", n_frames=7, width=64, height=48)
    cfg = _cfg(Method.dense, 1)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    small = np.zeros(10, np.uint32)
    with pytest.raises(InvalidArgument, match="destination too small"):
        sim.push_frames_streamed(frames[:5], ts[:5], chunk=2, out=small)
    # the simulation completed: the call's events are still readable (24-B form, device unpack)
    lib = sim._lib
    n = int(len(concat(run_oracle_stream(oracle, cfg, frames[:5], ts[:5]))))
    buf = np.zeros(n, EVENT_DTYPE)
    assert lib.evsim_gpu_copy_events(sim._h, ctypes.c_void_p(buf.ctypes.data), n, 1) == 0
    assert_same_events(buf, concat(run_oracle_stream(oracle, cfg, frames[:5], ts[:5])))
    # and the stream state advanced
    rest = sim.push_frames(frames[5:], ts[5:]).events
    assert_same_events(rest, concat(run_oracle_stream(oracle, cfg, frames, ts)[5:]))
    assert len(exp) == n + len(rest)


def test_streamed_rejects_magnitude_and_bad_batches():
    frames, ts = scenes.generate("c2", n_frames=4, width=32, height=32)
    sim = Simulator(SimulatorConfig.from_c(make_config(Method.dense, n_interp=3, events_per_crossing=1)))
    with pytest.raises(InvalidArgument, match="magnitude"):
        sim.push_frames_streamed(frames, ts)
    sim = Simulator(SimulatorConfig.from_c(make_config(Method.dense, n_interp=3)))
    bad = ts.copy()
    bad[2] = bad[1]
    with pytest.raises(InvalidArgument, match="strictly increasing"):
        sim.push_frames_streamed(frames, bad)
    # rejected atomically: the stream is untouched
    p, t, o = sim.push_frames_streamed(frames, ts, chunk=3)
    assert o[-1] == p.size


@pytest.mark.parametrize("mode,chunk", [(1, 0), (0, 0), (1, 20), (0, 37)])
def test_streamed_long_dense_pipelined(oracle, mode, chunk):
    """Dense streamed calls long enough for flow sub-batches inside a chunk
    and for the cross-chunk overlap: 45 frames in one chunk
    (4 sub-batches) or in chunks of ~20 / ~37 frames."""
    frames, ts = scenes.generate("c2", n_frames=45, width=100, height=76)
    cfg = _cfg(Method.dense, mode)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    packed, seg_t, seg_off = sim.push_frames_streamed(frames, ts, chunk=chunk)
    assert_same_events(unpack_events(packed, seg_t, seg_off), exp)
