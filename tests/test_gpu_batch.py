"""GPU: batched pushes (evsim_gpu_push_frames) are bit-identical to the
reference's frame-by-frame Simulator::push_frame, for every method / mode,
batch size and batch boundary placement."""
import numpy as np
import pytest

from helpers import assert_same_events, concat, run_oracle_stream
from paper_2209_04634_b200 import Frame, InvalidArgument, SimulatorConfig, Simulator, scenes
from paper_2209_04634_b200.abi import Method, make_config

pytestmark = pytest.mark.gpu


def _cfgs():
    out = []
    for m in (Method.difference_only, Method.dense, Method.sparse):
        for mode in (0, 1):
            out.append((m, mode, 0, 1))
    out += [(Method.dense, 1, 1, 1), (Method.dense, 0, 0, 0), (Method.sparse, 1, 0, 0), (Method.sparse, 0, 1, 1),
            (Method.dense, 1, 0, 0)]
    return out


@pytest.mark.parametrize("m,mode,mag,incl", _cfgs())
@pytest.mark.parametrize("batch", [1, 3, 7, 40])
def test_batch_matches_oracle(oracle, m, mode, mag, incl, batch):
    frames, ts = scenes.generate("c2", n_frames=9, width=100, height=76)
    cfg = make_config(m, n_interp=5 if m != Method.difference_only else 0, contrast_mode=mode,
                      events_per_crossing=mag, include_endpoints=incl, c_pos_log=0.1, c_neg_log=-0.12,
                      selection_threshold=4)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    got = []
    for a in range(0, len(frames), batch):
        got.append(sim.push_frames(frames[a:a + batch], ts[a:a + batch]).events)
    assert_same_events(concat(got), exp)


def test_batch_after_single_pushes_and_reset(oracle):
    frames, ts = scenes.generate("c3", n_frames=8, width=96, height=64)
    cfg = make_config(Method.sparse, n_interp=6, contrast_mode=1, c_pos_log=0.15, c_neg_log=-0.15)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    got = [sim.push_frame(Frame.from_array(frames[0], ts[0])).events,
           sim.push_frame(Frame.from_array(frames[1], ts[1])).events,
           sim.push_frames(frames[2:6], ts[2:6]).events,
           sim.push_frame(Frame.from_array(frames[6], ts[6])).events,
           sim.push_frames(frames[7:8], ts[7:8]).events]
    assert_same_events(concat(got), exp)
    sim.reset()
    again = sim.push_frames(frames, ts).events
    assert_same_events(again, exp)


def test_batch_collision_timestamps(oracle):
    frames, _ = scenes.generate("c1", n_frames=5, width=48, height=40)
    ts = np.array([0, 5, 9, 12, 100], np.int64)  # dt < K: equal sub-interval stamps
    cfg = make_config(Method.dense, n_interp=10)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    assert_same_events(sim.push_frames(frames, ts).events, exp)


def test_batch_rejected_atomically():
    frames, ts = scenes.generate("c1", n_frames=4, width=32, height=24)
    sim = Simulator(SimulatorConfig.defaults(Method.dense))
    sim.push_frames(frames[:2], ts[:2])
    bad = ts[2:].copy()
    bad[1] = bad[0]
    with pytest.raises(InvalidArgument, match="strictly increasing"):
        sim.push_frames(frames[2:], bad)
    # state untouched: the good continuation still works and matches
    out = sim.push_frames(frames[2:], ts[2:])
    assert len(out) > 0


def test_full_sequence_one_batch_c2_log(oracle):
    """The bench's shape: a whole 640x480 sequence in one launch sequence."""
    frames, ts = scenes.generate("c2", n_frames=6)
    cfg = make_config(Method.dense, n_interp=10, contrast_mode=1, c_pos_log=0.2, c_neg_log=-0.2)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    assert_same_events(sim.push_frames(frames, ts).events, exp)


@pytest.mark.parametrize("mode,mag,incl", [(1, 0, 1), (0, 0, 1), (1, 1, 1), (0, 1, 0), (1, 0, 0)])
def test_pipelined_dense_push_matches_oracle(oracle, mode, mag, incl):
    """A dense push of >= 16 pairs runs its flow in sub-batches on a second
    stream, overlapping the previous sub-batch's chain;
    with stage timing on, the same push runs serially.  Both must equal the
    oracle bit for bit."""
    frames, ts = scenes.generate("c2", n_frames=41, width=100, height=76)
    cfg = make_config(Method.dense, n_interp=6, contrast_mode=mode, events_per_crossing=mag,
                      include_endpoints=incl, c_pos_log=0.1, c_neg_log=-0.12)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    for profiling in (False, True):
        sim = Simulator(SimulatorConfig.from_c(cfg))
        sim.set_profiling(profiling)
        got = [sim.push_frames(frames[:1], ts[:1]).events, sim.push_frames(frames[1:], ts[1:]).events]
        assert_same_events(concat(got), exp, what=f"profiling={profiling}")


@pytest.mark.parametrize("where", [9, 10, 39])
@pytest.mark.parametrize("mode", [0, 1])
def test_pipelined_push_with_one_colliding_pair(oracle, where, mode):
    """Sub-batched pushes (41 frames -> 4 flow sub-batches of 10 pairs) emit
    per sub-batch only when every link has its own timestamp; one pair with
    dt < K (equal sub-interval stamps, finalize's stable sort,
    simulate.cpp:36-40) at the last pair of a sub-batch, the first pair of the
    next, or the last pair of the push must switch that off.  Single mode."""
    frames, ts = scenes.generate("c2", n_frames=41, width=100, height=76)
    ts = ts.copy()
    gap = np.full(40, 33333, np.int64)
    gap[where] = 2 + (where % 2)  # 2-3 us < K = 7
    ts[1:] = np.cumsum(gap)
    cfg = make_config(Method.dense, n_interp=6, contrast_mode=mode, c_pos_log=0.1, c_neg_log=-0.12)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    got = [sim.push_frames(frames[:1], ts[:1]).events, sim.push_frames(frames[1:], ts[1:]).events]
    assert_same_events(concat(got), exp)
